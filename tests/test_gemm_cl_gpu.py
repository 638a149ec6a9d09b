"""Numerics of the cluster split-K projection (pm_gemm_cl, gemm_cl.cu): the
whole projection -- split-K reduction through distributed shared memory and
the fused epilogue -- in one kernel.  Checked against torch fp32 (TF32 off)
and against the unfused kernels; every (slices, clusters) plan gives the same
answer up to fp32 summation order, and a token's row is bit-identical alone
or inside a batch (batch invariance)."""
import numpy as np
import pytest
import torch

from paper_2605_02189_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"
torch.backends.cuda.matmul.allow_tf32 = False


def _lin(n_out, k, seed, scale=0.05):
    g = torch.Generator(device=DEV).manual_seed(seed)
    w = (torch.randn(n_out, k, generator=g, device=DEV) * scale).to(torch.bfloat16)
    return w, ops.Linear(w), g


def _x(m_cap, m, k, g):
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    return x


@pytest.mark.parametrize("n_out,k,m", [(256, 256, 3), (6144, 4096, 128), (4096, 4096, 64), (4096, 12288, 100),
                                       (24576, 4096, 16), (10240, 5120, 33), (512, 64, 1), (8192, 8192, 128)])
def test_cl_store_vs_fp32(n_out, k, m):
    w, lin, g = _lin(n_out, k, n_out + k + m)
    m_cap = 128
    x = _x(m_cap, m, k, g)
    maps = ops.activation_maps(x)
    want = x[:m].float() @ w.float().T
    y = torch.zeros(m_cap, n_out, device=DEV, dtype=torch.bfloat16)
    lin.cl(maps, m, ops.CL_EPI_STORE, m_cap=m_cap, out=y, ld_out=n_out)
    torch.cuda.synchronize()
    err = (y[:m].float() - want).abs().max().item()
    assert err <= 2 ** -8 * want.abs().max().item() + 1e-3, err
    assert (y[m:] == 0).all()
    # batch invariance: token 0 alone gives the bit-identical row
    y1 = torch.zeros_like(y)
    lin.cl(maps, 1, ops.CL_EPI_STORE, m_cap=m_cap, out=y1, ld_out=n_out)
    torch.cuda.synchronize()
    assert torch.equal(y1[0], y[0])


@pytest.mark.parametrize("S", [1, 2, 3, 4])
def test_cl_every_plan_agrees(S):
    """Every (slices, clusters) split sums the same products: fp32 results
    agree to summation-order rounding (RESID epilogue keeps fp32)."""
    n_out, k, m = 4096, 4096, 77
    w, lin, g = _lin(n_out, k, 7)
    m_cap = 128
    x = _x(m_cap, m, k, g)
    maps = ops.activation_maps(x)
    want = x[:m].float() @ w.float().T
    for nc in sorted({1, 3, 7, 16}):
        lin._cl = (S, nc)
        r = torch.zeros(m_cap, n_out, device=DEV)
        lin.cl(maps, m, ops.CL_EPI_RESID, m_cap=m_cap, resid=r)
        torch.cuda.synchronize()
        assert torch.allclose(r[:m], want, atol=2e-4, rtol=1e-4), (S, nc, (r[:m] - want).abs().max().item())
        assert (r[m:] == 0).all()


def test_cl_silu_interleaved():
    ffn, k, m = 1536, 512, 24
    g = torch.Generator(device=DEV).manual_seed(3)
    gate = (torch.randn(ffn, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    up = (torch.randn(ffn, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    w = torch.stack([gate, up], dim=1).reshape(2 * ffn, k).contiguous()
    x = _x(128, m, k, g)
    out = torch.zeros(128, ffn, device=DEV, dtype=torch.bfloat16)
    lin = ops.Linear(w)
    lin.cl(ops.activation_maps(x), m, ops.CL_EPI_SILU, m_cap=128, out=out, ld_out=ffn)
    torch.cuda.synchronize()
    want = torch.nn.functional.silu(x[:m].float() @ gate.float().T) * (x[:m].float() @ up.float().T)
    assert (out[:m].float() - want).abs().max().item() < 2 ** -8 * want.abs().max().item() + 1e-3


@pytest.mark.parametrize("n_out,k,m", [(4096, 4096, 128), (5120, 8192, 64), (256, 512, 5)])
def test_cl_resid_folded_norm_chain(n_out, k, m):
    """O-style RESID epilogue with the next norm folded: resid += x W^T,
    xn = bf16(resid * w), per-tile sums of squares; a consumer GEMM with
    rs = (ssq, d) then equals W2 . RMSNorm(resid) * w in fp32 to bf16
    storage precision."""
    w, lin, g = _lin(n_out, k, n_out + m)
    m_cap = 128
    x = _x(m_cap, m, k, g)
    nw = (1 + 0.1 * torch.randn(n_out, generator=g, device=DEV)).to(torch.bfloat16)
    r0 = torch.randn(m_cap, n_out, generator=g, device=DEV)
    r = r0.clone()
    xn = torch.zeros(m_cap, n_out, device=DEV, dtype=torch.bfloat16)
    ssq = torch.zeros(n_out // 128, m_cap, device=DEV)
    lin.cl(ops.activation_maps(x), m, ops.CL_EPI_RESID, m_cap=m_cap, resid=r, norm_w=nw, xn=xn, ssq_out=ssq)
    torch.cuda.synchronize()
    want_r = r0[:m] + x[:m].float() @ w.float().T
    assert torch.allclose(r[:m], want_r, atol=2e-4, rtol=1e-4)
    assert torch.equal(r[m:], r0[m:])
    assert torch.equal(xn[:m], (r[:m] * nw.float()).to(torch.bfloat16))
    tiles = (r[:m] ** 2).view(m, n_out // 128, 128).sum(-1).T
    assert torch.allclose(ssq[:, :m], tiles, rtol=1e-5, atol=1e-5)
    # consumer: a projection of the normalised rows
    n2 = 1024
    w2, lin2, _ = _lin(n2, n_out, 99)
    y = torch.zeros(m_cap, n2, device=DEV, dtype=torch.bfloat16)
    eps = 1e-6
    lin2.cl(ops.activation_maps(xn), m, ops.CL_EPI_STORE, m_cap=m_cap, out=y, ld_out=n2, rs=(ssq, n_out), eps=eps)
    torch.cuda.synchronize()
    h = r[:m] * torch.rsqrt((r[:m] ** 2).mean(-1, keepdim=True) + eps) * nw.float()
    want = h @ w2.float().T
    assert (y[:m].float() - want).abs().max().item() <= 2 ** -7 * want.abs().max().item()


@pytest.mark.parametrize("m,V,k", [(3, 4096, 256), (40, 4096, 512), (77, 151936, 512), (128, 128256, 256)])
def test_cl_logits_argmax(m, V, k):
    g = torch.Generator(device=DEV).manual_seed(5)
    w = (torch.randn(V, k, generator=g, device=DEV) * 0.2).to(torch.bfloat16)
    lin = ops.Linear(w)
    m_cap = 128
    x = _x(m_cap, m, k, g)
    ws = ops.GemmWorkspace(m_cap, 1, lin.n_units, lin.n_units, DEV)
    logits = torch.zeros(m_cap, V, device=DEV)
    ids = torch.zeros(m_cap, dtype=torch.int32, device=DEV)
    lin.cl(ops.activation_maps(x), m, ops.CL_EPI_LOGITS, m_cap=m_cap, out=logits, ld_out=V, ws=ws)
    ops.argmax_reduce(ws, lin.n_units, m, ids)
    torch.cuda.synchronize()
    want = x[:m].float() @ w.float().T
    assert torch.allclose(logits[:m], want, atol=1e-3, rtol=1e-4)
    assert torch.equal(ids[:m].long(), logits[:m].argmax(-1))
    # without the logits buffer the argmax is unchanged
    ids2 = torch.zeros_like(ids)
    lin.cl(ops.activation_maps(x), m, ops.CL_EPI_LOGITS, m_cap=m_cap, out=None, ld_out=V, ws=ws)
    ops.argmax_reduce(ws, lin.n_units, m, ids2)
    torch.cuda.synchronize()
    assert torch.equal(ids2[:m], ids[:m])


@pytest.mark.parametrize("H,Hkv,hd,k,m,qk_norm", [(32, 8, 128, 4096, 128, True), (8, 2, 64, 256, 5, True),
                                                 (64, 8, 128, 5120, 64, True), (64, 8, 128, 8192, 33, False)])
def test_cl_qkv_rope_matches_unfused(H, Hkv, hd, k, m, qk_norm):
    """CL_QKV_ROPE == bf16 GEMM store then pm_qkv_rope_append (q and the
    appended K/V within one bf16 rounding)."""
    g = torch.Generator(device=DEV).manual_seed(H + k + m)
    n_out = (H + 2 * Hkv) * hd
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = 128
    x = _x(m_cap, m, k, g)
    lin = ops.Linear(w)
    maps = ops.activation_maps(x)
    L_s, layer, max_blocks = 2, 1, 8
    n_blocks = m * 4 + 4
    pool_ref = torch.zeros(n_blocks * 16 * L_s * 2 * Hkv * hd, dtype=torch.bfloat16, device=DEV)
    pool_cl = torch.zeros_like(pool_ref)
    bt = torch.randperm(n_blocks, generator=torch.Generator().manual_seed(m))[: m * 4].view(m, 4).to(torch.int32)
    btab = torch.zeros(m_cap, max_blocks, dtype=torch.int32)
    btab[:m, :4] = bt
    btab = btab.to(DEV)
    pos = torch.zeros(m_cap, dtype=torch.int32)
    pos[:m] = torch.randint(0, 64, (m,), generator=torch.Generator().manual_seed(k)).to(torch.int32)
    pos = pos.to(DEV)
    rope = torch.randn(128, hd, generator=g, device=DEV)
    qn = kn = None
    if qk_norm:
        qn = (1 + 0.1 * torch.randn(hd, generator=g, device=DEV)).to(torch.bfloat16)
        kn = (1 + 0.1 * torch.randn(hd, generator=g, device=DEV)).to(torch.bfloat16)
    qkv = torch.zeros(m_cap, n_out, device=DEV, dtype=torch.bfloat16)
    q_ref = torch.zeros(m_cap, H, hd, device=DEV, dtype=torch.bfloat16)
    q_cl = torch.zeros_like(q_ref)
    lin.cl(maps, m, ops.CL_EPI_STORE, m_cap=m_cap, out=qkv, ld_out=n_out)
    ops.qkv_rope_append(qkv, q_ref, pool_ref, btab, pos, rope, qn, kn, m, H, Hkv, hd, layer, L_s, 1e-6)
    lin.cl(maps, m, ops.CL_EPI_QKV_ROPE, m_cap=m_cap, eps=1e-6,
           rope=dict(q_out=q_cl, pool=pool_cl, block_table=btab, positions=pos, rope=rope, qn_w=qn, kn_w=kn, H=H,
                     Hkv=Hkv, hd=hd, layer=layer, L_s=L_s))
    torch.cuda.synchronize()
    tol = 2 ** -7
    assert torch.allclose(q_cl.float(), q_ref.float(), atol=tol * q_ref.abs().max().item(), rtol=tol)
    assert torch.allclose(pool_cl.float(), pool_ref.float(), atol=tol * pool_ref.abs().max().item(), rtol=tol)
    assert (pool_cl != 0).sum() == (pool_ref != 0).sum()


def test_cl_plans_fit_one_wave():
    """The planner never launches more clusters than can be co-resident."""
    for U, kb in ((24, 64), (16, 64), (96, 64), (16, 192), (594, 64), (40, 80), (200, 80), (501, 128)):
        S, nc = ops.cl_plan(U, kb)
        assert 1 <= S <= 4 and 1 <= nc <= U
        assert nc <= ops.cl_max_clusters(2 * S)
