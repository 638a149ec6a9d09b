"""fp32 decoder forward in MATRIX form over whole teacher-forced sequences --
the checker for the sm_100a engine at real model shapes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The same semantics as
``forward_ref`` (one token at a time, numpy), restated so that a request's
prompt plus its fed decode tokens run as ONE causal pass: the logits the
engine produced when it decoded position p are the logits this pass gives at
position p.  Plain torch fp32 (TF32 off), so it runs on the CPU for the
golden checks and on the GPU for the real-shape engine tests (a torch fp32
reference of the floating-point forward -- nothing here is on the product
path).  Pinned against ``transformers`` 5.5.0 (``tests/golden/hf_*.npz``,
``tests/test_oracle_hf.py``).  Semantics followed (transformers 5.5.0, not
under /root/reference -- the reference has no model math):
  * RMSNorm              qwen3/modeling_qwen3.py:50-67, llama:53
  * rotate-half RoPE     qwen3:151-182 (cos/sin of the shared fp32 table)
  * GQA / eager softmax  qwen3:184-193 (repeat_kv), fp32 softmax
  * per-head q/k norm    qwen3:248-264 (before RoPE)
  * SwiGLU MLP           llama:171
Every request attends only to its own keys (causal within the request), so a
batched GPU result matching it is batch-invariant by construction.
"""
from __future__ import annotations

import numpy as np
import torch


def _rmsnorm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


class SeqModel:
    """hp: dict(d, H, Hkv, hd, qk_norm, eps); layers: list of dicts of 2-D
    weights in HF layout [out, in] (any dtype -- upcast to fp32 here):
    attn_norm, wq, wk, wv, wo, mlp_norm, w_gate, w_up, w_down (+ q_norm,
    k_norm); embed [V, d]; final_norm [d]; lm_head [V, d]; rope_tab
    [max_pos, hd] (cos | sin halves, models.rope_table)."""

    def __init__(self, hp, layers, embed, final_norm, lm_head, rope_tab, device="cpu", chunk_tokens=8192,
                 storage_bf16=False):
        """storage_bf16: also round to bf16 wherever the GPU path STORES a
        bf16 tensor (as ``forward_ref.RefModel(storage_bf16=True)``: norm
        outputs, q/k/v, cached K/V, attention output, SwiGLU activation) --
        the twin that separates kernel arithmetic from bf16 storage error.
        The default is the pure fp32 reference."""
        self.r = (lambda t: t.to(torch.bfloat16).to(torch.float32)) if storage_bf16 else (lambda t: t)
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
        self.hp, self.dev = hp, torch.device(device)
        f = lambda t: (torch.as_tensor(t) if not isinstance(t, torch.Tensor) else t).to(self.dev, torch.float32)
        self.layers = [{k: f(v) for k, v in w.items() if v is not None} for w in layers]
        self.embed, self.final_norm, self.lm_head = f(embed), f(final_norm), f(lm_head)
        rope = f(rope_tab)
        half = hp["hd"] // 2
        self.cos, self.sin = rope[:, :half], rope[:, half:]
        self.chunk_tokens = chunk_tokens

    # ------------------------------------------------------------------ pieces
    def _rope(self, x, pos):
        """x [T, heads, hd] at positions pos [T]."""
        half = x.shape[-1] // 2
        c, s = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    def _layer(self, li, x, segs, pos, caches):
        """One decoder layer over the concatenated new tokens ``x`` [T, d].
        ``segs``: list of (a, b) row ranges, one per request; ``caches[j][li]``
        = (K, V) [P, Hkv, hd] of request j's earlier positions (appended to)."""
        hp, w = self.hp, self.layers[li]
        H, Hkv, hd, eps = hp["H"], hp["Hkv"], hp["hd"], hp["eps"]
        T, R = x.shape[0], self.r
        h = R(_rmsnorm(x, w["attn_norm"], eps))
        q = R(h @ w["wq"].T).view(T, H, hd)
        k = R(h @ w["wk"].T).view(T, Hkv, hd)
        v = R(h @ w["wv"].T).view(T, Hkv, hd)
        if hp["qk_norm"]:
            q = _rmsnorm(q, w["q_norm"], eps)
            k = _rmsnorm(k, w["k_norm"], eps)
        q, k = R(self._rope(q, pos)), R(self._rope(k, pos))
        o = torch.empty(T, H, hd, device=self.dev)
        g = H // Hkv
        scale = 1.0 / float(np.sqrt(hd))
        for j, (a, b) in enumerate(segs):
            Kp, Vp = caches[j][li]
            K = torch.cat([Kp, k[a:b]]) if Kp is not None else k[a:b]
            V = torch.cat([Vp, v[a:b]]) if Vp is not None else v[a:b]
            caches[j][li] = (K, V)
            L, n = K.shape[0], b - a
            Kh = K.permute(1, 0, 2).repeat_interleave(g, dim=0)      # [H, L, hd]
            Vh = V.permute(1, 0, 2).repeat_interleave(g, dim=0)
            s = (q[a:b].permute(1, 0, 2) @ Kh.transpose(1, 2)) * scale   # [H, n, L]
            qpos = torch.arange(L - n, L, device=self.dev)[:, None]
            s = s.masked_fill(torch.arange(L, device=self.dev)[None, :] > qpos, float("-inf"))
            o[a:b] = (torch.softmax(s, dim=-1) @ Vh).permute(1, 0, 2)
        x = x + R(o).reshape(T, H * hd) @ w["wo"].T
        h = R(_rmsnorm(x, w["mlp_norm"], eps))
        return x + R(torch.nn.functional.silu(h @ w["w_gate"].T) * (h @ w["w_up"].T)) @ w["w_down"].T

    def _run(self, new_tokens, caches, want):
        """Run every request's ``new_tokens[j]`` after its cache; returns, per
        request, the logits at its new rows ``want[j]`` (indices into the new
        tokens) as an fp32 tensor on the device."""
        rows, segs, pos = [], [], []
        for j, toks in enumerate(new_tokens):
            P = 0 if caches[j][0][0] is None else caches[j][0][0].shape[0]
            a = len(rows)
            rows.extend(int(t) for t in toks)
            segs.append((a, len(rows)))
            pos.extend(range(P, P + len(toks)))
        x = self.embed[torch.tensor(rows, device=self.dev, dtype=torch.long)]
        posd = torch.tensor(pos, device=self.dev, dtype=torch.long)
        for li in range(len(self.layers)):
            x = self._layer(li, x, segs, posd, caches)
        out = []
        for j, (a, b) in enumerate(segs):
            sel = x[a:b][torch.as_tensor(want[j], device=self.dev, dtype=torch.long)]
            out.append(self.r(_rmsnorm(sel, self.final_norm, self.hp["eps"])) @ self.lm_head.T)
        return out

    def _groups(self, lengths):
        """Consecutive request groups of at most ``chunk_tokens`` tokens."""
        grp, tot = [], 0
        for j, n in enumerate(lengths):
            if grp and tot + n > self.chunk_tokens:
                yield grp
                grp, tot = [], 0
            grp.append(j)
            tot += n
        if grp:
            yield grp

    # ------------------------------------------------------------------ API
    @torch.no_grad()
    def teacher_forced(self, seqs, want, numpy=True):
        """seqs[j]: token ids of request j (prompt + fed decode tokens);
        want[j]: positions whose logits to return.  Returns a list of fp32
        arrays [len(want[j]), V] (numpy, or device tensors with
        ``numpy=False``) -- the logits of the NEXT token after each wanted
        position (what the engine emits when it decodes it)."""
        out = [None] * len(seqs)
        for grp in self._groups([len(s) for s in seqs]):
            caches = [[(None, None)] * len(self.layers) for _ in grp]
            res = self._run([seqs[j] for j in grp], caches, [want[j] for j in grp])
            for j, r in zip(grp, res):
                out[j] = r.cpu().numpy() if numpy else r
        return out

    @torch.no_grad()
    def greedy(self, prompts, n_gen, first=None):
        """Free-running greedy decode of every request: after the prompt, feed
        the argmax ``n_gen`` times (``first[j]``, if given, replaces the argmax
        of the prompt's last position -- the engine's prefill token).  Returns
        (ids [R, n_gen + 1] = the fed tokens then the last argmax, top-2
        margins [R, n_gen + 1] of the fp32 logits at each choice)."""
        R = len(prompts)
        ids = np.zeros((R, n_gen + 1), dtype=np.int64)
        margin = np.zeros((R, n_gen + 1), dtype=np.float64)
        for grp in self._groups([len(p) for p in prompts]):
            caches = [[(None, None)] * len(self.layers) for _ in grp]
            lg = self._run([prompts[j] for j in grp], caches, [[len(prompts[j]) - 1] for j in grp])
            for step in range(n_gen + 1):
                nxt = []
                for gi, j in enumerate(grp):
                    top = torch.topk(lg[gi][0], 2)
                    margin[j, step] = float(top.values[0] - top.values[1])
                    t = int(top.indices[0])
                    if step == 0 and first is not None:
                        t = int(first[j])
                    ids[j, step] = t
                    nxt.append([t])
                if step == n_gen:
                    break
                lg = self._run(nxt, caches, [[0]] * len(grp))
        return ids, margin
