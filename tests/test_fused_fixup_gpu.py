"""In-kernel split-K fixup (Linear.enable_fused, the single-lane engines'
path): every projection finishes its split units inside the GEMM kernel.
It must equal the post-kernel path bit for bit -- same partial-sum order,
same epilogue arithmetic, same RMSNorm reduction tree -- and leave its
per-unit and per-row counters at zero so the next launch (and a CUDA-graph
replay) starts clean.  Shapes: the decode projections of the bench configs
(Qwen3-8B C2, Qwen3-32B C3 stage, Llama-70B C4 stage) at their step rows,
plus small / padded / whole-unit edge cases, on 116 and 128 SMs."""
import pytest
import torch

from paper_2605_02189_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _pair(w, sms):
    """(post-kernel Linear, fused Linear) over the same weight."""
    a, b = ops.Linear(w), ops.Linear(w)
    a.sms = b.sms = sms
    b.enable_fused(DEV)
    return a, b


def _ws(m_cap, lin):
    return ops.GemmWorkspace(m_cap, ops.GemmWorkspace.floats_needed([lin], m_cap), lin.n_units, lin.n_units, DEV)


PLAIN = [  # name, n_out, k, m, epilogue, sms
    ("c3 gate/up silu", 2 * 25600, 5120, 48, ops.EPI_SILU_MUL, 116),
    ("c2 gate/up silu", 2 * 12288, 4096, 128, ops.EPI_SILU_MUL, 116),
    ("c3 down resid", 5120, 25600, 48, ops.EPI_RESID_ADD, 116),
    ("c4 O resid", 8192, 8192, 24, ops.EPI_RESID_ADD, 116),
    ("store", 6144, 4096, 77, ops.EPI_STORE_BF16, 128),
    ("pad rows", 640, 8192, 33, ops.EPI_STORE_BF16, 116),
    ("one row", 4096, 4096, 1, ops.EPI_STORE_BF16, 116),
    ("c3 lm_head", 151936, 5120, 48, ops.EPI_LOGITS_ARGMAX, 116),
    ("logits ragged", 30000, 1024, 50, ops.EPI_LOGITS_ARGMAX, 128),
]


@pytest.mark.parametrize("name,n_out,k,m,epi,sms", PLAIN, ids=[p[0] for p in PLAIN])
def test_fused_gemm_equals_post_kernels(name, n_out, k, m, epi, sms):
    g = torch.Generator(device=DEV).manual_seed(n_out + k + m)
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = 256
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    ref, fus = _pair(w, sms)
    maps = ops.activation_maps(x)
    ws_r, ws_f = _ws(m_cap, ref), _ws(m_cap, fus)
    width = n_out // 2 if epi == ops.EPI_SILU_MUL else n_out
    dt = torch.float32 if epi in (ops.EPI_RESID_ADD, ops.EPI_LOGITS_ARGMAX) else torch.bfloat16
    y0 = torch.randn(m_cap, width, generator=g, device=DEV).to(dt)
    y_r, y_f = y0.clone(), y0.clone()
    ids_r = torch.full((m_cap,), -1, dtype=torch.int32, device=DEV)
    ids_f = ids_r.clone()
    for rep in range(2):   # twice: the counters must be re-armed by the first launch
        ref(maps, m, epi, y_r, width, ws_r)
        fus(maps, m, epi, y_f, width, ws_f)
        if epi == ops.EPI_LOGITS_ARGMAX:
            ops.argmax_reduce(ws_r, ref.n_units, m, ids_r)
            ops.argmax_reduce(ws_f, fus.n_units, m, ids_f)
        torch.cuda.synchronize()
        assert torch.equal(y_f, y_r), (name, rep)
        assert torch.equal(ids_f, ids_r), (name, rep)
        assert (ws_f.fix_cnt == 0).all(), (name, rep)
    assert fus.launches(m) == 1


RESID = [  # name, d, k, m, sms
    ("c3 O", 5120, 8192, 48, 116), ("c3 down", 5120, 25600, 48, 116), ("c2 O", 4096, 4096, 128, 116),
    ("c4 down", 8192, 28672, 24, 116), ("c4 O 32 rows", 8192, 8192, 32, 116), ("small", 512, 256, 7, 128),
    ("no split", 512, 64, 16, 116),
]


@pytest.mark.parametrize("name,d,k,m,sms", RESID, ids=[r[0] for r in RESID])
def test_fused_resid_rmsnorm_equals_post_kernels(name, d, k, m, sms):
    """Residual bit-for-bit and the next RMSNorm bit-for-bit (the 128-thread
    norm plays rmsnorm_kernel's 256-thread reduction tree); row counters re-armed."""
    g = torch.Generator(device=DEV).manual_seed(d + k + m)
    w = (torch.randn(d, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = 256
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    nw = (1 + 0.1 * torch.randn(d, generator=g, device=DEV)).to(torch.bfloat16)
    ref, fus = _pair(w, sms)
    maps = ops.activation_maps(x)
    ws_r, ws_f = _ws(m_cap, ref), _ws(m_cap, fus)
    r0 = torch.randn(m_cap, d, generator=g, device=DEV)
    r_r, r_f = r0.clone(), r0.clone()
    xn_r = torch.zeros(m_cap, d, device=DEV, dtype=torch.bfloat16)
    xn_f = torch.zeros_like(xn_r)
    for rep in range(2):
        ref.resid_rmsnorm(maps, m, r_r, ws_r, nw, xn_r, 1e-6, split_norm=True)
        fus.resid_rmsnorm(maps, m, r_f, ws_f, nw, xn_f, 1e-6)
        torch.cuda.synchronize()
        assert torch.equal(r_f, r_r), (name, rep)
        assert torch.equal(xn_f[:m], xn_r[:m]), (name, rep)
        assert (ws_f.row_cnt == 0).all() and (ws_f.fix_cnt == 0).all(), (name, rep)


QKV = [  # name, H, Hkv, hd, k, m, qk_norm, sms
    ("c3 qwen3-32b", 64, 8, 128, 5120, 48, True, 116), ("c2 qwen3-8b", 32, 8, 128, 4096, 128, True, 116),
    ("c4 llama-70b", 64, 8, 128, 8192, 24, False, 116), ("hd64", 8, 2, 64, 256, 5, True, 128),
    ("whole units", 600, 20, 64, 128, 40, False, 116),
]


@pytest.mark.parametrize("name,H,Hkv,hd,k,m,qk_norm,sms", QKV, ids=[q[0] for q in QKV])
def test_fused_qkv_rope_equals_post_kernel(name, H, Hkv, hd, k, m, qk_norm, sms):
    """q and the appended K/V bit-identical to the QKV post kernel."""
    g = torch.Generator(device=DEV).manual_seed(H + k + m)
    n_out = (H + 2 * Hkv) * hd
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = 256
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    ref, fus = _pair(w, sms)
    maps = ops.activation_maps(x)
    ws_r, ws_f = _ws(m_cap, ref), _ws(m_cap, fus)
    L_s, layer, max_blocks = 2, 1, 8
    n_blocks = m * 4 + 4
    pool_r = torch.zeros(n_blocks * 16 * L_s * 2 * Hkv * hd, dtype=torch.bfloat16, device=DEV)
    pool_f = torch.zeros_like(pool_r)
    bt = torch.randperm(n_blocks, generator=torch.Generator().manual_seed(m))[: m * 4].view(m, 4).to(torch.int32)
    btab = torch.zeros(m, max_blocks, dtype=torch.int32)
    btab[:, :4] = bt
    btab = btab.to(DEV)
    pos = torch.randint(0, 64, (m,), generator=torch.Generator().manual_seed(k)).to(torch.int32).to(DEV)
    rope = torch.randn(128, hd, generator=g, device=DEV)
    qn = kn = None
    if qk_norm:
        qn = (1 + 0.1 * torch.randn(hd, generator=g, device=DEV)).to(torch.bfloat16)
        kn = (1 + 0.1 * torch.randn(hd, generator=g, device=DEV)).to(torch.bfloat16)
    q_r = torch.zeros(m, H, hd, device=DEV, dtype=torch.bfloat16)
    q_f = torch.zeros_like(q_r)
    s_r = torch.zeros(m_cap, n_out, device=DEV, dtype=torch.bfloat16)
    s_f = torch.zeros_like(s_r)
    for rep in range(2):
        ref.qkv_rope(maps, m, s_r, ws_r, q_r, pool_r, btab, pos, rope, qn, kn, H, Hkv, hd, layer, L_s, 1e-6)
        fus.qkv_rope(maps, m, s_f, ws_f, q_f, pool_f, btab, pos, rope, qn, kn, H, Hkv, hd, layer, L_s, 1e-6)
        torch.cuda.synchronize()
        assert torch.equal(q_f, q_r), (name, rep)
        assert torch.equal(pool_f, pool_r), (name, rep)
        assert (ws_f.fix_cnt == 0).all(), (name, rep)


@pytest.mark.parametrize("mode", ["fused", "poll"])
def test_fused_in_cuda_graph_replays(mode, monkeypatch):
    """A graph of back-to-back projections with programmatic dependent launch
    -- in-kernel fixups (counters shared through one workspace), or polling
    post kernels (one counter slice per call site: a polling post kernel may
    start before the previous projection's post kernel re-armed its counts)
    -- replays to the same result as eager grid-wait launches."""
    g = torch.Generator(device=DEV).manual_seed(5)
    d, ffn, m, m_cap = 5120, 25600, 48, 256
    w_o = (torch.randn(d, 8192, generator=g, device=DEV) * 0.02).to(torch.bfloat16)
    w_gu = (torch.randn(2 * ffn, d, generator=g, device=DEV) * 0.02).to(torch.bfloat16)
    w_dn = (torch.randn(d, ffn, generator=g, device=DEV) * 0.02).to(torch.bfloat16)
    nw = (1 + 0.1 * torch.randn(d, generator=g, device=DEV)).to(torch.bfloat16)
    attn = torch.zeros(m_cap, 8192, device=DEV, dtype=torch.bfloat16)
    attn[:m] = torch.randn(m, 8192, generator=g, device=DEV).to(torch.bfloat16)
    resid0 = torch.randn(m_cap, d, generator=g, device=DEV)
    outs = []
    for fused in (False, True):
        monkeypatch.setattr(ops, "FIX_POLL_ON", fused and mode == "poll")
        lins = [ops.Linear(w) for w in (w_o, w_gu, w_dn)]
        for lin in lins:
            lin.sms = 116
            if fused and mode == "fused":
                lin.enable_fused(DEV)
        ws = ops.GemmWorkspace(m_cap, ops.GemmWorkspace.floats_needed(lins, m_cap), max(l.n_units for l in lins), 1, DEV,
                               sites=3)
        resid = resid0.clone()
        xn = torch.zeros(m_cap, d, device=DEV, dtype=torch.bfloat16)
        act = torch.zeros(m_cap, ffn, device=DEV, dtype=torch.bfloat16)
        xm, am, atm = ops.activation_maps(xn), ops.activation_maps(act), ops.activation_maps(attn)
        st = torch.cuda.Stream()

        def chain():
            lins[0].resid_rmsnorm(atm, m, resid, ws, nw, xn, 1e-6, st, split_norm=True, site=0)
            lins[1](xm, m, ops.EPI_SILU_MUL, act, ffn, ws, st, site=1)
            lins[2].resid_rmsnorm(am, m, resid, ws, nw, xn, 1e-6, st, split_norm=True, site=2)
        if fused:
            with torch.cuda.stream(st):
                chain()   # warm-up (attributes)
            torch.cuda.synchronize()
            resid.copy_(resid0)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                chain()
            for _ in range(3):
                with torch.cuda.stream(st):
                    resid.copy_(resid0)
                    gr.replay()
                torch.cuda.synchronize()
        else:
            with torch.cuda.stream(st):
                chain()
            torch.cuda.synchronize()
        outs.append((resid.clone(), xn[:m].clone(), act[:m].clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("name,n_out,k,m,epi,sms", PLAIN, ids=[p[0] for p in PLAIN])
def test_polling_post_kernels_equal_grid_wait(name, n_out, k, m, epi, sms, monkeypatch):
    """FIX_POLL (post-kernel CTAs start on their unit's arrivals) == FIX_POST
    (post kernel waits for the whole GEMM grid), bit for bit, counters re-armed."""
    g = torch.Generator(device=DEV).manual_seed(n_out + k + m + 1)
    w = (torch.randn(n_out, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = 256
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    maps = ops.activation_maps(x)
    width = n_out // 2 if epi == ops.EPI_SILU_MUL else n_out
    dt = torch.float32 if epi in (ops.EPI_RESID_ADD, ops.EPI_LOGITS_ARGMAX) else torch.bfloat16
    y0 = torch.randn(m_cap, width, generator=g, device=DEV).to(dt)
    outs = []
    for poll in (False, True):
        monkeypatch.setattr(ops, "FIX_POLL_ON", poll)
        lin = ops.Linear(w)
        lin.sms = sms
        ws = _ws(m_cap, lin)
        y = y0.clone()
        ids = torch.full((m_cap,), -1, dtype=torch.int32, device=DEV)
        for _ in range(2):
            lin(maps, m, epi, y, width, ws)
            if epi == ops.EPI_LOGITS_ARGMAX:
                ops.argmax_reduce(ws, lin.n_units, m, ids)
        torch.cuda.synchronize()
        assert (ws.fix_cnt == 0).all()
        outs.append((y.cpu(), ids.cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("split_norm", [False, True])
@pytest.mark.parametrize("name,d,k,m,sms", RESID[:4], ids=[r[0] for r in RESID[:4]])
def test_polling_resid_norm_and_qkv_equal_grid_wait(name, d, k, m, sms, split_norm, monkeypatch):
    g = torch.Generator(device=DEV).manual_seed(d + k + m + 3)
    w = (torch.randn(d, k, generator=g, device=DEV) * 0.05).to(torch.bfloat16)
    m_cap = 256
    x = torch.zeros(m_cap, k, device=DEV, dtype=torch.bfloat16)
    x[:m] = torch.randn(m, k, generator=g, device=DEV).to(torch.bfloat16)
    nw = (1 + 0.1 * torch.randn(d, generator=g, device=DEV)).to(torch.bfloat16)
    maps = ops.activation_maps(x)
    r0 = torch.randn(m_cap, d, generator=g, device=DEV)
    outs = []
    for poll in (False, True):
        monkeypatch.setattr(ops, "FIX_POLL_ON", poll)
        lin = ops.Linear(w)
        lin.sms = sms
        ws = _ws(m_cap, lin)
        r = r0.clone()
        xn = torch.zeros(m_cap, d, device=DEV, dtype=torch.bfloat16)
        for _ in range(2):
            lin.resid_rmsnorm(maps, m, r, ws, nw, xn, 1e-6, split_norm=split_norm)
        torch.cuda.synchronize()
        assert (ws.fix_cnt == 0).all() and (ws.row_cnt == 0).all()
        outs.append((r.cpu(), xn[:m].cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
