"""Diagnostic: run one decode token of the TINY model op by op on the GPU and
compare every intermediate with the numpy twin (bf16 storage points)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import forward_ref as ref  # noqa: E402
from paper_2605_02189_b200 import ops  # noqa: E402
from paper_2605_02189_b200.models import TINY, rope_table  # noqa: E402
from paper_2605_02189_b200.stage import StageExecutor  # noqa: E402

s = TINY
dev = torch.device("cuda")
ex = StageExecutor(s, range(s.layers), first=True, last=True, m_cap=16, pool_blocks=8, max_blocks=4,
                   n_slots=4, device=dev, keep_logical=True, max_pos=64)
ex.enable_logits()
M = 1
ex.tok_table[0] = 123
ex.block_table[0, 0] = 3
ex.positions[0] = 0
ex.seq_lens[0] = 1
ex.slots[0] = 0
R = ref.bf16
tab = rope_table(s, 64)


def cmp(name, gpu, want):
    g = gpu.float().cpu().numpy().reshape(want.shape)
    e = np.abs(g - want).max()
    print(f"{name:12s} max|x|={np.abs(want).max():.4g} err={e:.3g} rel={e / max(np.abs(want).max(), 1e-30):.3g}")


x = ex.embed[123].float().cpu().numpy()
ops.embed(ex.tok_table, ex.slots, ex.embed, ex.resid, M)
cmp("embed", ex.resid[0], x)
for li, w in enumerate(ex.W):
    L = {k: v.float().cpu().numpy() for k, v in ex.logical[li].items()}
    ops.rmsnorm(ex.resid, w["attn_norm"], ex.xn, M, s.eps)
    h = R(ref.rmsnorm(x, L["attn_norm"], s.eps))
    cmp(f"L{li} xn", ex.xn[0], h)
    w["qkv"](ex.xn_maps, M, ops.EPI_STORE_BF16, ex.qkv, s.qkv_out, ex.gws)
    wqkv = np.concatenate([L["wq"], L["wk"], L["wv"]], 0)
    qkv = R(wqkv @ h)
    cmp(f"L{li} qkv", ex.qkv[0], qkv)
    ops.qkv_rope_append(ex.qkv, ex.q, ex.pool, ex.block_table, ex.positions, ex.rope, w["q_norm"],
                        w["k_norm"], M, s.H, s.Hkv, s.hd, li, ex.L_s, s.eps)
    q = R(ref.rope(qkv[:s.H * s.hd].reshape(s.H, s.hd), 0, tab))
    cmp(f"L{li} q", ex.q[0], q)
    ops.paged_attention(ex.pool_map, ex.q, ex.block_table, ex.seq_lens, ex.attn, ex.aws,
                        M, s.H, s.Hkv, s.hd, li, ex.L_s)
    k = R(ref.rope(qkv[s.H * s.hd:(s.H + s.Hkv) * s.hd].reshape(s.Hkv, s.hd), 0, tab))
    v = qkv[(s.H + s.Hkv) * s.hd:].reshape(s.Hkv, s.hd)
    o = R(ref.attend(q, k[None], v[None], s.H // s.Hkv))
    cmp(f"L{li} attn", ex.attn[0], o)
    ops.Linear  # noqa
    w["o"](ex.attn_maps, M, ops.EPI_RESID_ADD, ex.resid, s.d, ex.gws)
    x = x + L["wo"] @ o.reshape(-1)
    cmp(f"L{li} resid1", ex.resid[0], x)
    ops.rmsnorm(ex.resid, w["mlp_norm"], ex.xn, M, s.eps)
    h = R(ref.rmsnorm(x, L["mlp_norm"], s.eps))
    cmp(f"L{li} xn2", ex.xn[0], h)
    w["gu"](ex.xn_maps, M, ops.EPI_SILU_MUL, ex.act, s.ffn, ex.gws)
    a = R(ref.silu(L["w_gate"] @ h) * (L["w_up"] @ h))
    cmp(f"L{li} act", ex.act[0], a)
    w["down"](ex.act_maps, M, ops.EPI_RESID_ADD, ex.resid, s.d, ex.gws)
    x = x + L["w_down"] @ a
    cmp(f"L{li} resid2", ex.resid[0], x)
ops.rmsnorm(ex.resid, ex.final_norm, ex.xn, M, s.eps)
h = R(ref.rmsnorm(x, ex.final_norm.float().cpu().numpy(), s.eps))
cmp("final xn", ex.xn[0], h)
ex.lm_head(ex.xn_maps, M, ops.EPI_LOGITS_ARGMAX, ex.logits, s.vocab, ex.gws)
cmp("logits", ex.logits[0], ex.lm_head_logical.float().cpu().numpy() @ h)
torch.cuda.synchronize()
