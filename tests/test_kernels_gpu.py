"""Numerics of each sm_100a kernel against plain references (torch fp32 for
the GEMM, the fp32 numpy oracle for norm / RoPE / paged attention) and
bit-exact checks of where the KV-append lands in the block-first pool."""
import math

import numpy as np
import pytest
import torch

from oracle import forward_ref as ref
from paper_2605_02189_b200 import ops
from paper_2605_02189_b200.models import LLAMA3_70B, QWEN3_32B, QWEN3_8B, TINY, rope_table

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _ws(m_cap, lin):
    return ops.GemmWorkspace(m_cap, ops.GemmWorkspace.floats_needed([lin], m_cap), lin.n_units, lin.n_units, DEV)


@pytest.mark.parametrize("n_out,k,m", [
    (256, 256, 8), (512, 768, 16), (6144, 4096, 128), (1024, 12288, 64),
    (384, 1024, 200), (256, 512, 300), (128, 64, 1), (4096, 4096, 32), (24576, 4096, 256), (640, 8192, 100)])
def test_gemm_store_and_resid(n_out, k, m):
    g = torch.Generator(device=DEV).manual_seed(n_out + k + m)
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = max(256, m)
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    lin = ops.Linear(w)
    maps = ops.activation_maps(x)
    ws = _ws(m_cap, lin)
    want = x[:m].float() @ w.float().T
    y = torch.zeros(m_cap, n_out, device=DEV, dtype=torch.bfloat16)
    lin(maps, m, ops.EPI_STORE_BF16, y, n_out, ws)
    torch.cuda.synchronize()
    err = (y[:m].float() - want).abs().max().item()
    assert err <= 2e-2 * max(1.0, want.abs().max().item()), err
    assert (y[m:] == 0).all()
    r0 = torch.randn(m_cap, n_out, generator=g, device=DEV)
    r = r0.clone()
    lin(maps, m, ops.EPI_RESID_ADD, r, n_out, ws)
    torch.cuda.synchronize()
    assert torch.allclose(r[:m], r0[:m] + want, atol=1e-3, rtol=1e-4)
    assert torch.equal(r[m:], r0[m:])
    # batch invariance (one token tile): token 0 alone gives the bit-identical row
    if m <= 256:
        y1 = torch.zeros_like(y)
        lin(maps, 1, ops.EPI_STORE_BF16, y1, n_out, ws)
        torch.cuda.synchronize()
        assert torch.equal(y1[0], y[0])


def test_gemm_silu_mul_interleaved():
    ffn, k, m = 384, 512, 24
    g = torch.Generator(device=DEV).manual_seed(3)
    gate = (torch.randn(ffn, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    up = (torch.randn(ffn, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    w = torch.stack([gate, up], dim=1).reshape(2 * ffn, k).contiguous()  # row 2i gate_i, 2i+1 up_i
    x = torch.zeros(256, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    out = torch.zeros(256, ffn, device=DEV, dtype=torch.bfloat16)
    lin = ops.Linear(w)
    lin(ops.activation_maps(x), m, ops.EPI_SILU_MUL, out, ffn, _ws(256, lin))
    torch.cuda.synchronize()
    gg, uu = x[:m].float() @ gate.float().T, x[:m].float() @ up.float().T
    want = torch.nn.functional.silu(gg) * uu
    assert (out[:m].float() - want).abs().max().item() < 2e-2 * want.abs().max().item() + 1e-3


@pytest.mark.parametrize("m,V,k", [(3, 4096, 256), (40, 4096, 256), (77, 151936, 512)])
def test_gemm_logits_argmax(m, V, k):
    g = torch.Generator(device=DEV).manual_seed(5)
    w = (torch.randn(V, k, generator=g, device=DEV) * 0.2).to(torch.bfloat16)
    x = torch.zeros(256, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    lin = ops.Linear(w)
    ws = _ws(256, lin)
    logits = torch.zeros(256, V, device=DEV)
    lin(ops.activation_maps(x), m, ops.EPI_LOGITS_ARGMAX, logits, V, ws)
    ids = torch.full((256,), -1, dtype=torch.int32, device=DEV)
    ops.argmax_reduce(ws, lin.n_units, m, ids)
    torch.cuda.synchronize()
    want = x[:m].float() @ w.float().T
    assert torch.allclose(logits[:m], want, atol=1e-3, rtol=1e-3)
    assert torch.equal(ids[:m].long(), logits[:m].argmax(dim=1))


def test_rmsnorm_and_embed():
    d, M = 4096, 37
    g = torch.Generator(device=DEV).manual_seed(7)
    table = torch.randn(1000, d, generator=g, device=DEV).to(torch.bfloat16)
    ids = torch.randint(0, 1000, (M,), generator=g, device=DEV, dtype=torch.int32)
    resid = torch.empty(M, d, device=DEV)
    ops.embed(ids, None, table, resid, M)
    w = (1 + 0.1 * torch.randn(d, generator=g, device=DEV)).to(torch.bfloat16)
    y = torch.empty(M, d, device=DEV, dtype=torch.bfloat16)
    ops.rmsnorm(resid, w, y, M, 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(resid, table[ids.long()].float())
    want = ref.rmsnorm(resid.cpu().numpy(), w.float().cpu().numpy(), 1e-6)
    np.testing.assert_allclose(y.float().cpu().numpy(), want, atol=2e-2, rtol=1e-2)


def _pool(n_blocks, L_s, Hkv, hd):
    return torch.zeros(n_blocks * 16 * L_s * 2 * Hkv * hd, dtype=torch.bfloat16, device=DEV)


@pytest.mark.parametrize("garbage,kv5", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("spec", [TINY, QWEN3_8B, QWEN3_32B, LLAMA3_70B])   # GQA groups 2, 4, 8, 8
def test_rope_append_and_paged_attention(spec, garbage, kv5):
    """Random prefixes scattered over random physical blocks; the current
    token goes through the fused qk-norm/RoPE/append kernel, then attention
    reads the whole prefix through the block table.  garbage: every slot not
    written holds NaN bits (a recycled pool allocation) -- the rows' partial
    last blocks must not leak them into the output."""
    rng = np.random.default_rng(11)
    H, Hkv, hd, L_s, layer = spec.H, spec.Hkv, spec.hd, 3, 1
    lens = [1, 15, 16, 17, 100, 255, 256, 257, 700, 1025]  # prefix BEFORE this token
    M = len(lens)
    max_blocks = 72
    n_blocks = sum((L + 1 + 15) // 16 for L in lens) + 5
    perm = rng.permutation(n_blocks)
    tables = np.zeros((M, max_blocks), np.int32)
    cur = 0
    for r, L in enumerate(lens):
        nb = (L + 1 + 15) // 16
        tables[r, :nb] = perm[cur:cur + nb]
        cur += nb
    pool = _pool(n_blocks, L_s, Hkv, hd)
    if garbage:
        pool.view(torch.int16).fill_(-1)   # 0xffff: bf16 NaN
    P = pool.view(n_blocks, 16, L_s, 2, Hkv, hd)
    # existing prefix KV for positions < L (random, written through the table)
    hist_k = [rng.standard_normal((L, Hkv, hd)).astype(np.float32) for L in lens]
    hist_v = [rng.standard_normal((L, Hkv, hd)).astype(np.float32) for L in lens]
    Pc = P.cpu()
    for r, L in enumerate(lens):
        for p in range(L):
            b = tables[r, p // 16]
            Pc[b, p % 16, layer, 0] = torch.from_numpy(hist_k[r][p]).to(torch.bfloat16)
            Pc[b, p % 16, layer, 1] = torch.from_numpy(hist_v[r][p]).to(torch.bfloat16)
    P.copy_(Pc)
    hist_k = [torch.from_numpy(h).to(torch.bfloat16).float().numpy() for h in hist_k]
    hist_v = [torch.from_numpy(h).to(torch.bfloat16).float().numpy() for h in hist_v]
    qkv = torch.from_numpy(rng.standard_normal((M, spec.qkv_out)).astype(np.float32)).to(torch.bfloat16).to(DEV)
    rope = torch.from_numpy(rope_table(spec, 2048)).to(DEV)
    qn = kn = None
    if spec.qk_norm:
        qn = (1 + 0.1 * torch.randn(hd, device=DEV)).to(torch.bfloat16)
        kn = (1 + 0.1 * torch.randn(hd, device=DEV)).to(torch.bfloat16)
    q_out = torch.empty(M, H, hd, dtype=torch.bfloat16, device=DEV)
    bt = torch.from_numpy(tables).to(DEV)
    pos = torch.tensor(lens, dtype=torch.int32, device=DEV)
    ops.qkv_rope_append(qkv, q_out, pool, bt, pos, rope, qn, kn, M, H, Hkv, hd, layer, L_s, spec.eps)
    aws = ops.AttnWorkspace(M, Hkv, hd, max_blocks, DEV)
    out = torch.empty(M, H, hd, dtype=torch.bfloat16, device=DEV)
    seq = pos + 1
    tmap = ops.pool_tmap(pool, L_s, Hkv, hd, kv5=kv5)   # 2-D boxes or the 5-D one-copy map
    aws.set_work([L + 1 for L in lens])
    # decode=garbage: the NaN-pool cases also load each row's older blocks ahead of the
    # dependency wait on qkv_rope_append (cfg bit 5), the others after it
    ops.paged_attention(tmap, q_out, bt, seq, out, aws, M, H, Hkv, hd, layer, L_s, decode=garbage)
    torch.cuda.synchronize()
    assert (aws.counters == 0).all()
    tab = rope_table(spec, 2048)
    x = qkv.float().cpu().numpy()
    Pn = P.float().cpu().numpy()
    for r, L in enumerate(lens):
        q = x[r, :H * hd].reshape(H, hd)
        k = x[r, H * hd:(H + Hkv) * hd].reshape(Hkv, hd)
        v = x[r, (H + Hkv) * hd:].reshape(Hkv, hd)
        if spec.qk_norm:
            q = ref.rmsnorm(q, qn.float().cpu().numpy(), spec.eps)
            k = ref.rmsnorm(k, kn.float().cpu().numpy(), spec.eps)
        q, k = ref.rope(q, L, tab), ref.rope(k, L, tab)
        np.testing.assert_allclose(q_out[r].float().cpu().numpy(), q, atol=3e-2, rtol=1e-2)
        b, s = tables[r, L // 16], L % 16
        np.testing.assert_allclose(Pn[b, s, layer, 0], k, atol=3e-2, rtol=1e-2)
        assert np.array_equal(Pn[b, s, layer, 1], torch.from_numpy(v).to(torch.bfloat16).float().numpy())
        # attention uses the bf16 values actually stored / produced
        K = np.concatenate([hist_k[r], Pn[b, s, layer, 0][None]], 0)
        V = np.concatenate([hist_v[r], Pn[b, s, layer, 1][None]], 0)
        want = ref.attend(q_out[r].float().cpu().numpy(), K, V, H // Hkv)
        got = out[r].float().cpu().numpy()
        np.testing.assert_allclose(got, want, atol=2e-2, rtol=2e-2, err_msg=f"row {r} len {L}")
    assert np.isfinite(out.float().cpu().numpy()).all()
    # untouched layers / slots stay as they were
    if not garbage:
        assert np.all(Pn[:, :, 0] == 0) and np.all(Pn[:, :, 2] == 0)


@pytest.mark.parametrize("n_out,k,m", [(4096, 4096, 128), (512, 256, 7), (8192, 1024, 200), (512, 64, 16),
                                       (4096, 12288, 64)])
@pytest.mark.parametrize("split_norm", [False, True])
def test_fused_resid_rmsnorm_matches_unfused(n_out, k, m, split_norm):
    """pm_gemm_resid_rmsnorm == pm_gemm(+resid) then pm_rmsnorm: the residual
    bit-for-bit, the normalised row bit-for-bit (same reduction order), and
    the per-row arrival counters re-armed; (512, 64) splits no unit and takes
    the separate-norm path, as does split_norm=True."""
    g = torch.Generator(device=DEV).manual_seed(n_out + k + m)
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = max(256, m)
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    nw = (1 + 0.1 * torch.randn(n_out, generator=g, device=DEV)).to(torch.bfloat16)
    lin = ops.Linear(w)
    maps = ops.activation_maps(x)
    ws = _ws(m_cap, lin)
    r0 = torch.randn(m_cap, n_out, generator=g, device=DEV)
    r_ref, r_fused = r0.clone(), r0.clone()
    xn_ref = torch.zeros(m_cap, n_out, device=DEV, dtype=torch.bfloat16)
    xn_fused = torch.zeros_like(xn_ref)
    lin(maps, m, ops.EPI_RESID_ADD, r_ref, n_out, ws)
    ops.rmsnorm(r_ref, nw, xn_ref, m, 1e-6)
    lin.resid_rmsnorm(maps, m, r_fused, ws, nw, xn_fused, 1e-6, split_norm=split_norm)
    torch.cuda.synchronize()
    assert torch.equal(r_fused, r_ref)
    assert torch.equal(xn_fused[:m], xn_ref[:m])
    assert (ws.row_cnt == 0).all()


@pytest.mark.parametrize("H,Hkv,hd,k,m,qk_norm", [(32, 8, 128, 4096, 128, True), (8, 2, 64, 256, 5, True),
                                                 (600, 20, 64, 128, 40, False)])
def test_fused_qkv_rope_matches_unfused(H, Hkv, hd, k, m, qk_norm):
    """pm_gemm_qkv_rope == pm_gemm(store bf16) then pm_qkv_rope_append: q and
    the appended K/V agree to one bf16 rounding (the per-head norm sums in a
    different order); (600, 20, 64, k=128) leaves units whole."""
    g = torch.Generator(device=DEV).manual_seed(H + k + m)
    n_out = (H + 2 * Hkv) * hd
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = 256
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    lin = ops.Linear(w)
    maps = ops.activation_maps(x)
    ws = _ws(m_cap, lin)
    L_s, layer, max_blocks = 2, 1, 8
    n_blocks = m * 4 + 4
    pool_ref = torch.zeros(n_blocks * 16 * L_s * 2 * Hkv * hd, dtype=torch.bfloat16, device=DEV)
    pool_fused = torch.zeros_like(pool_ref)
    bt = torch.randperm(n_blocks, generator=torch.Generator().manual_seed(m))[: m * 4].view(m, 4).to(torch.int32)
    btab = torch.zeros(m, max_blocks, dtype=torch.int32)
    btab[:, :4] = bt
    btab = btab.to(DEV)
    pos = torch.randint(0, 64, (m,), generator=torch.Generator().manual_seed(k)).to(torch.int32).to(DEV)
    spec_rope = torch.randn(128, hd, generator=g, device=DEV)
    qn = kn = None
    if qk_norm:
        qn = (1 + 0.1 * torch.randn(hd, generator=g, device=DEV)).to(torch.bfloat16)
        kn = (1 + 0.1 * torch.randn(hd, generator=g, device=DEV)).to(torch.bfloat16)
    qkv = torch.zeros(m_cap, n_out, device=DEV, dtype=torch.bfloat16)
    q_ref = torch.zeros(m, H, hd, device=DEV, dtype=torch.bfloat16)
    q_fused = torch.zeros_like(q_ref)
    lin(maps, m, ops.EPI_STORE_BF16, qkv, n_out, ws)
    ops.qkv_rope_append(qkv, q_ref, pool_ref, btab, pos, spec_rope, qn, kn, m, H, Hkv, hd, layer, L_s, 1e-6)
    scratch = torch.zeros_like(qkv)
    lin.qkv_rope(maps, m, scratch, ws, q_fused, pool_fused, btab, pos, spec_rope, qn, kn, H, Hkv, hd, layer, L_s,
                 1e-6)
    torch.cuda.synchronize()
    tol = 2 ** -7  # one bf16 rounding step (relative)
    assert torch.allclose(q_fused.float(), q_ref.float(), atol=tol * q_ref.abs().max().item(), rtol=tol)
    assert torch.allclose(pool_fused.float(), pool_ref.float(), atol=tol * pool_ref.abs().max().item(), rtol=tol)
    assert (pool_fused != 0).sum() == (pool_ref != 0).sum()
