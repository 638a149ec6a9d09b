"""fp32 numpy decode forward -- the checker for the sm_100a kernels.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  PARITY UNPINNED by the
reference: the reference package has no weights, no forward and no token
values.  This restates the third-party HF semantics
(transformers 5.5.0, not under /root/reference):
  * RMSNorm            models/llama/modeling_llama.py:53 / qwen3:50-67
                       y = w * (x * rsqrt(mean(x^2) + eps))
  * rotate-half RoPE   llama:146, qwen3:151-182
  * GQA                qwen3:184-193 (repeat_kv)
  * q/k per-head norm  qwen3:248-264 (before RoPE)
  * SwiGLU MLP         llama:171  down(silu(gate(x)) * up(x))
Every request is run UNBATCHED (one sequence at a time, its own KV), so a
batched GPU result that matches it is batch-invariant by construction.  All
math is fp32 on the bf16-rounded weights; the RoPE table is the shared fp32
table from ``rope_table`` (computed in float64, rounded once).
"""
import numpy as np


def rmsnorm(x, w, eps):
    x = x.astype(np.float32)
    return (x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + np.float32(eps))) * w


def rope(x, pos, table):
    """x [..., hd] at integer position(s) pos (broadcast over leading dims)."""
    hd = x.shape[-1]
    half = hd // 2
    cs = table[pos]
    cos, sin = cs[..., :half], cs[..., half:]
    if np.ndim(pos) and x.ndim == 3:  # [B, heads, hd] with pos [B]
        cos, sin = cos[:, None, :], sin[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)


def bf16(x):
    """Round fp32 -> bf16 (round-to-nearest-even) and back, in numpy."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def silu(x):
    return x / (1.0 + np.exp(-x))


def attend(q, k, v, group):
    """q [H, hd]; k, v [L, Hkv, hd] -> [H, hd] (softmax(q k^T / sqrt(hd)) v)."""
    H, hd = q.shape
    out = np.empty_like(q)
    for h in range(H):
        g = h // group
        s = (k[:, g, :] @ q[h]) / np.float32(np.sqrt(hd))
        p = np.exp(s - s.max())
        out[h] = (p / p.sum()) @ v[:, g, :]
    return out


class RefModel:
    """hp: dict(d, layers, H, Hkv, hd, ffn, vocab, qk_norm, eps); layers: list
    of dicts of fp32 arrays (HF layout [out, in]); embed, final_norm, lm_head."""

    def __init__(self, hp, layers, embed, final_norm, lm_head, rope_tab, storage_bf16=False):
        """storage_bf16: also round to bf16 wherever the GPU path STORES a bf16
        tensor (norm outputs, qkv, q, cached k/v, attention output, SwiGLU
        activation) -- a diagnostic twin that isolates kernel arithmetic from
        bf16 storage error.  The default is the pure fp32 reference."""
        self.r = bf16 if storage_bf16 else (lambda x: x)
        self.hp = hp
        self.layers = layers
        self.embed = embed
        self.final_norm = final_norm
        self.lm_head = lm_head
        self.rope = rope_tab

    def new_cache(self):
        return [([], []) for _ in self.layers]

    def layer_step(self, li, x, pos, cache):
        """One token of one request through layer li; x [d] fp32; cache list of (K, V)."""
        hp, w = self.hp, self.layers[li]
        H, Hkv, hd, eps = hp["H"], hp["Hkv"], hp["hd"], hp["eps"]
        R = self.r
        h = R(rmsnorm(x, w["attn_norm"], eps))
        q = R(w["wq"] @ h).reshape(H, hd)
        k = R(w["wk"] @ h).reshape(Hkv, hd)
        v = R(w["wv"] @ h).reshape(Hkv, hd)
        if hp["qk_norm"]:
            q = rmsnorm(q, w["q_norm"], eps)
            k = rmsnorm(k, w["k_norm"], eps)
        q = R(rope(q, pos, self.rope))
        k = R(rope(k, pos, self.rope))
        cache[0].append(k)
        cache[1].append(v)
        o = R(attend(q, np.stack(cache[0]), np.stack(cache[1]), H // Hkv))
        x = x + w["wo"] @ o.reshape(-1)
        h = R(rmsnorm(x, w["mlp_norm"], eps))
        return x + w["w_down"] @ R(silu(w["w_gate"] @ h) * (w["w_up"] @ h))

    def token_step(self, tok, pos, caches):
        """Embed one token at position pos, run all layers; returns logits [V]."""
        x = self.embed[tok].astype(np.float32)
        for li in range(len(self.layers)):
            x = self.layer_step(li, x, pos, caches[li])
        return self.lm_head @ self.r(rmsnorm(x, self.final_norm, self.hp["eps"]))

    def run_request(self, prompt, n_gen, forced=None):
        """Teacher-force the prompt, then decode n_gen tokens.  If ``forced``
        is given, those tokens are fed instead of the argmax (teacher-forced
        decode).  Returns (logits of each decode step [n_gen, V], greedy ids)."""
        caches = self.new_cache()
        logits = None
        for p, tok in enumerate(prompt):
            logits = self.token_step(int(tok), p, caches)
        outs, ids = [], []
        nxt = int(np.argmax(logits))
        for s in range(n_gen):
            tok = nxt if forced is None else int(forced[s])
            ids.append(nxt)
            logits = self.token_step(tok, len(prompt) + s, caches)
            outs.append(logits)
            nxt = int(np.argmax(logits))
        return np.stack(outs), ids, caches
