"""Tensor-level wrappers over the C-ABI kernels (torch for device memory and
streams only).  Every op runs a hand-written sm_100a kernel from
``libpmb200.so``; there is no eager/PyTorch fallback."""

from __future__ import annotations

import ctypes as C
import math

import torch

from . import _C

SMS = 148
BM, BK = 128, 64


class KernelTimer:
    """Optional per-launch CUDA-event timing (bench.py's roofline leg): events
    are recorded on the launching stream around each kernel, with the
    launch's algorithmic HBM bytes."""

    def __init__(self):
        self.pending = []   # (kind, bytes, start_ev, end_ev, mid_ev or None)

    def around(self, kind, nbytes, stream, fn, split=False):
        """``split``: a GEMM call -- an extra event between its main kernel
        and its fixup kernel (pm_gemm_split_event) times them separately."""
        s = stream if stream is not None else torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        mid = torch.cuda.Event(enable_timing=True) if split else None
        a.record(s)
        if mid is not None:
            mid.record(s)   # create the event; re-recorded after the main kernel
            _C.call("pm_gemm_split_event", C.c_void_p(mid.cuda_event))
        fn()
        b.record(s)
        self.pending.append((kind, nbytes, a, b, mid))

    def summary(self):
        out = {}
        for kind, nbytes, a, b, mid in self.pending:
            d = out.setdefault(kind, {"launches": 0, "bytes": 0, "seconds": 0.0})
            d["launches"] += 1
            d["bytes"] += nbytes
            if mid is not None:
                d["seconds"] += a.elapsed_time(mid) * 1e-3
                p = out.setdefault(kind + "_fixup", {"launches": 0, "bytes": 0, "seconds": 0.0})
                p["launches"] += 1
                p["seconds"] += mid.elapsed_time(b) * 1e-3
            else:
                d["seconds"] += a.elapsed_time(b) * 1e-3
        return out


TIMER = None  # set to a KernelTimer to time every launch


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class TensorMap:
    """A 64-byte-aligned host copy of a CUtensorMap (passed by value to the
    kernels).  Keeps the described tensor alive."""

    def __init__(self, tensor, inner, outer, row_stride_bytes, box_inner, box_outer, swizzle=True):
        self._raw = (C.c_ubyte * 192)()
        addr = C.addressof(self._raw)
        self.addr = (addr + 63) & ~63
        self.tensor = tensor
        _C.call("pm_tmap_encode_2d", C.c_void_p(self.addr), C.c_void_p(tensor.data_ptr()),
                inner, outer, row_stride_bytes, box_inner, box_outer, 1 if swizzle else 0)

    @property
    def ptr(self):
        return C.c_void_p(self.addr)


def matrix_tmap(t: torch.Tensor, box_rows: int) -> TensorMap:
    """K-major bf16 matrix [rows, K] -> TMA map with a [box_rows x 64] box."""
    assert t.dtype == torch.bfloat16 and t.dim() == 2 and t.stride(1) == 1
    return TensorMap(t, t.shape[1], t.shape[0], t.stride(0) * 2, BK, box_rows)


def bn_for(m_tok: int) -> int:
    for bn in (16, 32, 64, 128, 256):
        if m_tok <= bn:
            return bn
    return 256


EPI_STORE_BF16, EPI_RESID_ADD, EPI_SILU_MUL, EPI_LOGITS_ARGMAX = 0, 1, 2, 3
# how split stream-K units are finished (pm_gemm's fix_mode): post kernel after the
# whole GEMM grid / in-kernel tasks / post kernel polling per-unit arrivals.
# FIX_POLL is opt-in (PM_FIX_POLL=1) and NOT for CUDA-graph replays: eager launches
# are bit-identical to FIX_POST (tests/test_fused_fixup_gpu.py) and the per-stage
# benches gain ~0.5-1 %, but engine steps replayed from CUDA graphs with programmatic
# dependent launch produce wrong logits (correct with graphs and PDL off, or eager
# with PDL on) -- profiles/r2/fused_fixup.md.
FIX_POST, FIX_FUSED, FIX_POLL = 0, 1, 2
FIX_POLL_ON = __import__("os").environ.get("PM_FIX_POLL", "0") == "1"
UNIT_ROWS = 256


def pack_weight(w: torch.Tensor):
    """[N, K] bf16 (K-major) -> [N_pad/256][K/64][2][128][64] with every
    128x64 tile in the 128B-swizzled K-major UMMA shared-memory image
    (16-byte chunk c of row r stored at chunk c ^ (r % 8)), so the GEMM moves
    one contiguous 32 KB chunk per pipeline stage with a plain bulk copy.
    Rows are zero-padded to a multiple of 256."""
    n, k = w.shape
    assert k % BK == 0
    n_pad = -(-n // UNIT_ROWS) * UNIT_ROWS
    if n_pad != n:
        w = torch.cat([w, torch.zeros(n_pad - n, k, dtype=w.dtype, device=w.device)])
    kb = k // BK
    src = w.view(n_pad // UNIT_ROWS, 2, 128, kb, 8, 8).permute(0, 3, 1, 2, 4, 5)  # unit,kb,half,row,chunk,e
    out = torch.empty(n_pad // UNIT_ROWS, kb, 2, 128, 8, 8, dtype=w.dtype, device=w.device)
    for rr in range(8):
        perm = torch.tensor([c ^ rr for c in range(8)], device=w.device)
        out[:, :, :, rr::8] = src[:, :, :, rr::8].index_select(4, perm)
    return out, n_pad // UNIT_ROWS


PAIR_MAX_UNITS = int(__import__("os").environ.get("PM_PAIR_MAX_UNITS", "64"))   # narrower projections run on 2-CTA clusters (measured: QKV/O/down win, gate/up loses)


# SMs a decode GEMM's stream-K workers span.  Measured on the C2 bench
# (two lanes in flight, round 2, tools/ab_tune*.sh): 136 -> 5.50-5.55 ms/step,
# 140 -> 5.55, 144 -> 5.80-5.85, 128 -> 5.81-5.88, 132 -> 5.96, 148 slower
# still -- the other lane's fixup / attention CTAs start on the free SMs
# instead of queueing behind the GEMM's drain (PM_GEMM_CTAS overrides).
GEMM_CTAS = int(__import__("os").environ.get("PM_GEMM_CTAS", "136"))
# ... and with a single micro-batch in flight (per-stage runs): measured C3
# 2.140 -> 2.122 ms/step at 116 (PM_GEMM_CTAS_1LANE overrides)
GEMM_CTAS_1LANE = int(__import__("os").environ.get("PM_GEMM_CTAS_1LANE", "116"))


def gemm_plan(n_units: int, kb: int, m_tok: int, sms: int = None):
    """Stream-K geometry of one launch: (bn, grid CTAs, max segments per
    unit, token tiles, pair).  Narrow projections (fewer than
    PAIR_MAX_UNITS 256-row units) use 2-CTA cluster workers -- each CTA
    computes one 128-row half and the pair shares one multicast activation
    tile, which halves every split segment's partial and the number of
    segments; wide ones use one CTA per worker.  The k-block ranges depend on
    (units, K, #SMs) only -- not on m_tok for m_tok <= 256 -- which keeps
    results batch-invariant."""
    sms = GEMM_CTAS if sms is None else sms
    bn = bn_for(m_tok)
    tt = -(-m_tok // bn)
    total = n_units * tt * kb
    pair = n_units < PAIR_MAX_UNITS
    per = 2 if pair else 1
    workers = min(sms // per, total)
    import os
    if os.environ.get("PM_GEMM_GRID"):  # tuning experiments only (must match the library's override)
        workers = min(int(os.environ["PM_GEMM_GRID"]) // per, total)
    segs = _C.lib().pm_gemm_max_segments(total, kb, workers)
    return bn, per * workers, segs, tt, pair


# ---------------------------------------------------------------- cluster split-K GEMM (gemm_cl.cu)
import os as _os

# The cluster path finishes every projection (split-K reduction + epilogue)
# inside one kernel; with PM_GEMM_CL=1 steps of up to CL_MAX_M rows use it.
# Default OFF: measured slower than stream-K + fixup at C2 (QKV 27.9 vs 16.4
# us, tools/gemm_cl_bench.py): each CTA's weight stream tops out near 42 GB/s
# when a 128-row half shares SM ingress with a full activation tile, and the
# owner-phase reduction is latency-bound (profiles/r2/gemm_cl_*.txt).
CL_GEMM = _os.environ.get("PM_GEMM_CL", "0") == "1"
CL_MAX_M = 128
CL_EPI_STORE, CL_EPI_SILU, CL_EPI_RESID, CL_EPI_LOGITS, CL_EPI_QKV_ROPE = 0, 1, 2, 3, 4
# CTAs a cluster launch may span, and the per-SM weight-streaming rate the
# planner assumes (bytes/s); tuning knobs
CL_CTAS = int(_os.environ.get("PM_CL_CTAS", "148"))
CL_SM_BPS = float(_os.environ.get("PM_CL_SM_GBPS", "60")) * 1e9
CL_HBM_BPS = 6.5e12
CL_UNIT_S = 0.6e-6          # per-unit reduction/epilogue latency not hidden behind the next unit
_CL_MAX_ACTIVE_FALLBACK = {2: 74, 4: 33, 6: 22, 8: 15}   # measured on B200 (no GPU: planner tests)
_cl_active = {}


def cl_max_clusters(cluster_size: int) -> int:
    """Co-resident clusters of ``cluster_size`` CTAs (the 128-token
    instantiation, the largest shared-memory footprint)."""
    v = _cl_active.get(cluster_size)
    if v is None:
        if torch.cuda.is_available():
            _C.call("pm_prepare_gemm_cl")   # the smem attribute the occupancy query depends on
            out = C.c_int(0)
            _C.call("pm_gemm_cl_max_clusters", 128, cluster_size, C.byref(out))
            v = int(out.value)
        else:
            v = _CL_MAX_ACTIVE_FALLBACK[cluster_size]
        _cl_active[cluster_size] = v
    return v


def cl_plan(n_units: int, kb: int, ctas: int = None):
    """(slices S, clusters NC) of a cluster split-K launch: the choice that
    minimises the modelled time max(busiest CTA's weight bytes / per-SM rate,
    all weight bytes / HBM rate) + per-unit reduction latency, over S in 1..4
    and NC co-resident clusters of 2S CTAs.  Depends on (units, K) only --
    never on the token count -- so results are batch-invariant."""
    ctas = CL_CTAS if ctas is None else ctas
    best, best_t = None, None
    total = n_units * kb * 2 * CL_BK_BYTES
    for S in (1, 2, 3, 4):
        if S > kb:
            continue
        cs = 2 * S
        nc_max = min(n_units, cl_max_clusters(cs), ctas // cs)
        for nc in range(1, nc_max + 1):
            units = -(-n_units // nc)
            per_cta = units * -(-kb // S) * CL_BK_BYTES
            t = max(per_cta / CL_SM_BPS, total / CL_HBM_BPS) + units * CL_UNIT_S
            key = (round(t * 1e8), nc * cs)
            if best_t is None or key < best_t:
                best, best_t = (S, nc), key
    if best is None:
        raise RuntimeError(f"no co-resident cluster plan for {n_units} units x {kb} k-blocks")
    return best


CL_BK_BYTES = 128 * BK * 2   # one 128x64 bf16 weight tile
_cl_part = {}
_cl_prepared = False


def cl_scratch(device) -> torch.Tensor:
    """fp32 split-K partial scratch of the cluster GEMM: one [128 x 128]
    slot per CTA of the largest launch.  Shared by every launch on the device:
    each kernel writes its slots only after its programmatic-launch wait, i.e.
    after the previous kernel on its stream finished; kernels of different
    streams (lanes) get their own via ``cl_scratch_for``."""
    return cl_scratch_for(device, 0)


def cl_scratch_for(device, lane: int) -> torch.Tensor:
    key = (str(device), lane)
    t = _cl_part.get(key)
    if t is None:
        t = _cl_part[key] = torch.empty(CL_CTAS_MAX * 128 * 128, dtype=torch.float32, device=device)
    return t


CL_CTAS_MAX = 160


class GemmWorkspace:
    """Stream-K partials, per-row counters and argmax partials shared by all
    projections of one executor (launches on one stream run in order)."""

    def __init__(self, m_cap: int, ws_floats: int, max_units: int, vocab_units: int, device, sites: int = 1):
        self.m_cap = m_cap
        self.ws = torch.empty(max(1, ws_floats), dtype=torch.float32, device=device)
        # one argmax tile per 128-row half of a vocabulary unit
        self.amax_val = torch.empty(2 * max(1, vocab_units) * m_cap, dtype=torch.float32, device=device)
        self.amax_idx = torch.empty(2 * max(1, vocab_units) * m_cap, dtype=torch.int32, device=device)
        # per-row arrival counts of the fused residual + RMSNorm epilogue; kernels leave them zero
        self.row_cnt = torch.zeros(m_cap, dtype=torch.int32, device=device)
        # per-unit segment arrivals + readers / finished tasks of FIX_POLL / FIX_FUSED launches; left
        # zero.  One slice per GEMM call site of a step (``sites``): a polling post kernel may start
        # before the previous projection's post kernel has re-armed ITS counts, so consecutive
        # projections must not share a slice
        self.fix_stride = 2 * max(1, max_units, vocab_units)
        self.fix_cnt = torch.zeros(self.fix_stride * max(1, sites), dtype=torch.int32, device=device)

    def fix_ptr(self, site: int = 0):
        assert 0 <= site < self.fix_cnt.numel() // self.fix_stride, "GEMM call site out of range"
        return C.c_void_p(self.fix_cnt.data_ptr() + 4 * self.fix_stride * site)

    @staticmethod
    def floats_needed(linears, m_cap):
        need = 1
        for lin in linears:
            for m in sorted({min(m_cap, x) for x in (16, 32, 64, 128, 256, m_cap)}):
                bn, grid, segs, tt, _pair = gemm_plan(lin.n_units, lin.kb, m, lin.sms)
                need = max(need, lin.n_units * tt * segs * bn * UNIT_ROWS)
        return need


class Linear:
    """One projection: packed weight + stream-K launch plans."""

    def __init__(self, weight: torch.Tensor):
        assert weight.is_contiguous() and weight.dtype == torch.bfloat16
        self.n_out, self.k = weight.shape
        self.kb = self.k // BK
        self.packed, self.n_units = pack_weight(weight)
        self.weight_bytes = self.n_out * self.k * 2
        self._plans = {}
        self.sms = None   # SMs the stream-K workers span (None: GEMM_CTAS)
        self._cl = None   # (slices, clusters) of the cluster split-K launch (cl_plan)
        self.cl_ctas = None
        # in-kernel split-K fixup (single-lane engines, see pm_gemm): the task unit lists
        self.fused = False
        self._fix = None

    def enable_fused(self, device):
        """Finish split units inside the GEMM kernel from now on (one stream of
        dependent kernels only: the kernel waits on its own CTAs).  Builds the
        task-unit lists -- the split units, and every unit for the QKV post --
        which depend on (units, K, workers) only."""
        import numpy as np
        bn, grid, segs, tt, pair = self.plan(1)
        workers = grid // 2 if pair else grid
        buf = np.zeros(self.n_units, dtype=np.int32)
        n = _C.lib().pm_gemm_fix_units(C.c_longlong(self.n_units * self.kb), self.kb, workers,
                                       buf.ctypes.data_as(C.c_void_p))
        split = torch.from_numpy(buf[:n].copy()).to(device)
        every = torch.arange(self.n_units, dtype=torch.int32, device=device)
        self._fix = {False: (split, n), True: (every, self.n_units)}
        self.fused = True

    def _fixargs(self, m_tok, ws, qkv=False, site=0):
        """(mode, counters, unit list, count) of a launch: the in-kernel fixup
        when fused (one token tile), else the post kernels polling per-unit
        arrivals (FIX_POLL) unless PM_FIX_POLL=0."""
        if self.fused and self.plan(m_tok)[3] == 1:
            lst, n = self._fix[qkv]
            return FIX_FUSED, ws.fix_ptr(site), C.c_void_p(lst.data_ptr()), n
        if FIX_POLL_ON and self.plan(m_tok)[3] == 1:   # counters sized for one token tile
            return FIX_POLL, ws.fix_ptr(site), None, 0
        return FIX_POST, None, None, 0

    def launches(self, m_tok) -> int:
        """Kernels one call launches: the stream-K GEMM, plus gemm_reduce when
        the partition splits units (none when the fixup is in-kernel)."""
        if self.fused and self.plan(m_tok)[3] == 1:
            return 1
        return 1 + (self.plan(m_tok)[2] > 1)

    def plan(self, m_tok):
        p = self._plans.get(m_tok)
        if p is None:
            p = self._plans[m_tok] = gemm_plan(self.n_units, self.kb, m_tok, self.sms)
        return p

    @staticmethod
    def _pf(prefetch):
        """(ptr, bytes, span): prefetch = (tensor, bytes) for the contiguous
        first bytes, or (tensor, bytes, span) for one stripe per CTA spread
        over ``span`` bytes (the next GEMM's workers' first k-blocks)."""
        if prefetch is None:
            return None, 0, 0
        return C.c_void_p(prefetch[0].data_ptr()), int(prefetch[1]), int(prefetch[2]) if len(prefetch) > 2 else 0

    def _timed(self, kind_bytes, stream, go):
        if TIMER is None:
            go()
        else:
            TIMER.around("gemm", kind_bytes, stream, go, split=True)

    def __call__(self, x_maps: dict, m_tok: int, epilogue: int, out, ld_out: int, ws: GemmWorkspace,
                 stream=None, prefetch=None, site: int = 0):
        """``prefetch``: optional (tensor, nbytes) the next operation reads
        first; the kernel pulls it into L2 while it drains."""
        bn, grid, segs, tt, pair = self.plan(m_tok)
        pf_ptr, pf_bytes, pf_span = self._pf(prefetch)
        fx = self._fixargs(m_tok, ws, site=site)

        def go():
            _C.call("pm_gemm", _ptr(self.packed), x_maps[bn // 2 if pair else bn].ptr, self.n_out, self.n_units, self.k, m_tok, bn,
                    grid, int(pair), epilogue, _ptr(out), ld_out, _ptr(ws.ws), segs,
                    _ptr(ws.amax_val), _ptr(ws.amax_idx), ws.m_cap, pf_ptr, pf_bytes, pf_span, *fx, _stream(stream))
        out_b = {EPI_STORE_BF16: 2, EPI_RESID_ADD: 8, EPI_SILU_MUL: 1,
                 EPI_LOGITS_ARGMAX: 4 if out is not None else 0}[epilogue]
        self._timed(self.weight_bytes + m_tok * self.k * 2 + m_tok * self.n_out * out_b, stream, go)

    def resid_rmsnorm(self, x_maps: dict, m_tok: int, resid, ws: GemmWorkspace, norm_w, xn, eps: float,
                      stream=None, prefetch=None, split_norm: bool = False, site: int = 0):
        """resid += x W^T, then xn = RMSNorm(resid) * norm_w -- the residual
        projection fused with the next layer norm (pm_gemm_resid_rmsnorm)."""
        bn, grid, segs, tt, pair = self.plan(m_tok)
        pf_ptr, pf_bytes, pf_span = self._pf(prefetch)
        fx = self._fixargs(m_tok, ws, site=site)

        def go():
            _C.call("pm_gemm_resid_rmsnorm", _ptr(self.packed), x_maps[bn // 2 if pair else bn].ptr, self.n_out, self.n_units, self.k,
                    m_tok, bn, grid, int(pair), _ptr(resid), _ptr(ws.ws), segs, ws.m_cap, pf_ptr, pf_bytes, pf_span, _ptr(norm_w),
                    _ptr(xn), float(eps), _ptr(ws.row_cnt), int(split_norm), *fx, _stream(stream))
        self._timed(self.weight_bytes + m_tok * self.k * 2 + m_tok * self.n_out * (8 + 4 + 2), stream, go)

    def cl(self, x_maps: dict, m_tok: int, epilogue: int, stream=None, *, m_cap: int, out=None, ld_out=0, rs=None, eps=0.0,
           resid=None, norm_w=None, xn=None, ssq_out=None, ws: GemmWorkspace = None, rope=None, part=None):
        """Cluster split-K launch (pm_gemm_cl): the whole projection incl. its
        epilogue in one kernel.  ``rs`` = (ssq tensor, d_in): the input rows
        are bf16(x * w) of a folded RMSNorm (scale every token column by
        rsqrt(mean(x^2) + eps)); ``rope`` = dict(q_out, pool, block_table,
        positions, rope, qn_w, kn_w, H, Hkv, hd, layer, L_s) for the QKV
        epilogue; LOGITS writes the argmax tiles of ``ws``.  ``m_cap``: the row
        capacity of the activation / ssq / argmax buffers (their row stride).
        ``part``: the split-K partial scratch (cl_scratch_for; one per stream
        that may run GEMMs concurrently)."""
        assert m_tok <= CL_MAX_M
        bn = bn_for(m_tok)
        global _cl_prepared
        if not _cl_prepared:
            _C.call("pm_prepare_gemm_cl")
            _cl_prepared = True
        if self._cl is None:
            self._cl = cl_plan(self.n_units, self.kb, self.cl_ctas)
        S, nc = self._cl
        ssq_in, n_ht, d_in = (None, 0, 0) if rs is None else (rs[0], rs[1] // 128, rs[1])
        r = rope or {}
        amax_v, amax_i = (ws.amax_val, ws.amax_idx) if epilogue == CL_EPI_LOGITS else (None, None)
        _C.call("pm_gemm_cl", _ptr(self.packed), x_maps[bn // 2].ptr, self.n_out, self.n_units, self.k, m_tok, bn,
                m_cap, S, nc, epilogue, _ptr(out), ld_out, _ptr(ssq_in), n_ht, d_in, float(eps), _ptr(resid),
                _ptr(norm_w), _ptr(xn), _ptr(ssq_out), _ptr(amax_v), _ptr(amax_i), _ptr(r.get("q_out")),
                _ptr(r.get("pool")), _ptr(r.get("block_table")), _ptr(r.get("positions")), _ptr(r.get("rope")),
                _ptr(r.get("qn_w")), _ptr(r.get("kn_w")), r.get("H", 0), r.get("Hkv", 0), r.get("hd", 0),
                r.get("layer", 0), r.get("L_s", 0), r["block_table"].shape[1] if rope else 0, _ptr(part if part is not None else cl_scratch(self.packed.device)),
                _stream(stream))

    def qkv_rope(self, x_maps: dict, m_tok: int, qkv, ws: GemmWorkspace, q_out, pool, block_table, positions,
                 rope, qn_w, kn_w, H, Hkv, hd, layer, L_s, eps, stream=None, prefetch=None, site: int = 0):
        """QKV projection fused with q/k RMSNorm + RoPE + paged KV append
        (pm_gemm_qkv_rope); ``qkv`` is scratch for units left whole."""
        bn, grid, segs, tt, pair = self.plan(m_tok)
        pf_ptr, pf_bytes, pf_span = self._pf(prefetch)
        fx = self._fixargs(m_tok, ws, qkv=True, site=site)

        def go():
            _C.call("pm_gemm_qkv_rope", _ptr(self.packed), x_maps[bn // 2 if pair else bn].ptr, self.n_out, self.n_units, self.k,
                    m_tok, bn, grid, int(pair), _ptr(qkv), _ptr(ws.ws), segs, ws.m_cap, pf_ptr, pf_bytes, pf_span, *fx, _ptr(q_out),
                    _ptr(pool), _ptr(block_table), _ptr(positions), _ptr(rope), _ptr(qn_w), _ptr(kn_w), H, Hkv,
                    hd, layer, L_s, block_table.shape[1], float(eps), _stream(stream))
        self._timed(self.weight_bytes + m_tok * self.k * 2 + m_tok * self.n_out * 2, stream, go)


def activation_maps(buf: torch.Tensor) -> dict:
    """TMA maps of an activation buffer [m_cap, K] with a [rows x 64] box for
    every token tile BN and half tile BN / 2 (each CTA of a GEMM pair loads
    half the tile and multicasts it)."""
    return {rows: matrix_tmap(buf, rows) for rows in (8, 16, 32, 64, 128, 256)}


def embed(tok_table, slots, table, resid, M, stream=None):
    _C.call("pm_embed", _ptr(tok_table), _ptr(slots), _ptr(table), _ptr(resid), M, table.shape[1], _stream(stream))


def rmsnorm(x, w, y, M, eps, stream=None):
    _C.call("pm_rmsnorm", _ptr(x), _ptr(w), _ptr(y), M, x.shape[-1], eps, _stream(stream))


def qkv_rope_append(qkv, q_out, pool, block_table, positions, rope, qn_w, kn_w, M, H, Hkv, hd, layer,
                    L_s, eps, stream=None):
    _C.call("pm_qkv_rope_append", _ptr(qkv), _ptr(q_out), _ptr(pool), _ptr(block_table), _ptr(positions),
            _ptr(rope), _ptr(qn_w), _ptr(kn_w), M, H, Hkv, hd, layer, L_s, block_table.shape[1], eps,
            _stream(stream))


ATTN_KV5 = int(_os.environ.get("PM_ATTN_KV5", "0"))   # 5-D pool map: A/B measured neutral-to-slower at C2


class PoolMap(TensorMap):
    """pm_tmap_encode_pool's 5-D map of the block-first pool: one TMA copy
    moves a KV block's K and V of one (layer, kv head)."""

    def __init__(self, pool, n_rows, L_s, Hkv, hd):
        self._raw = (C.c_ubyte * 192)()
        self.addr = (C.addressof(self._raw) + 63) & ~63
        self.tensor = pool
        _C.call("pm_tmap_encode_pool", C.c_void_p(self.addr), C.c_void_p(pool.data_ptr()), n_rows, L_s, Hkv, hd)


def pool_tmap(pool: torch.Tensor, L_s: int, Hkv: int, hd: int, kv5: bool = None) -> TensorMap:
    """TMA map of the block-first pool for pm_paged_attention: the 2-D view
    rows = block*16 + slot, cols = (layer, k|v, head, dim) with a 16 slots x 64
    dims box, 128B swizzle (four copies per KV block; default), or the 5-D map
    (one copy per block; ``kv5`` / PM_ATTN_KV5=1)."""
    n_rows = pool.numel() // (L_s * 2 * Hkv * hd)
    width = L_s * 2 * Hkv * hd
    if ATTN_KV5 if kv5 is None else kv5:
        return PoolMap(pool, n_rows, L_s, Hkv, hd)
    return TensorMap(pool, width, n_rows, width * 2, 64, 16)


# Balanced attention work split (pm_attn_work_list): every (row, kv head)'s KV
# blocks are laid end to end and cut into one contiguous range per warp, then
# into pieces of at most ATTN_MAXP blocks (the kernel's per-piece block-id
# slots); a warp gets at least ATTN_MINQ blocks (bounds the pieces, i.e. the
# merge work, of one (row, head) when the step is small).
ATTN_MAXP = 32
ATTN_MINQ = 16


def attn_max_chunks(max_blocks: int) -> int:
    """Pieces one (row, head) of up to ``max_blocks`` blocks can be cut into."""
    return -(-max_blocks // ATTN_MAXP) + -(-max_blocks // ATTN_MINQ) + 1


def attn_work_len(m_cap: int, hkv: int, max_blocks: int, workers: int) -> int:
    """Ints a work list for up to m_cap rows can take (3 + warps + 4 per piece)."""
    units = m_cap * hkv
    pieces = 2 * units + workers + -(-units * max_blocks // ATTN_MAXP)
    return 6 + workers + 4 * pieces


class AttnWorkspace:
    """Per-piece partials [M][Hkv][chunks][8][hd] + (m, l), merge counters and the work list."""

    def __init__(self, m_cap, Hkv, hd, max_blocks, device, cfg=None, rows_hint=None):
        """``rows_hint``: the rows a step usually carries (a micro-batch), which
        sizes the launch-configuration choice; default ``m_cap``."""
        self.Hkv = Hkv
        cuda = torch.cuda.is_available()
        if cfg is None:
            cfg = choose_attn_cfg(rows_hint or m_cap, Hkv, hd, max_blocks) if cuda else -1
        self.cfg = cfg
        self.workers = _C.lib().pm_attn_workers_cfg(hd, cfg) if cuda else 0
        self.max_chunks = attn_max_chunks(max_blocks)
        self.o = torch.empty(m_cap * Hkv * self.max_chunks * 8 * hd, dtype=torch.float32, device=device)
        self.ml = torch.empty(m_cap * Hkv * self.max_chunks * 16, dtype=torch.float32, device=device)
        self.counters = torch.zeros(m_cap * Hkv, dtype=torch.int32, device=device)
        # the step's balanced work list (attn_work_list), uploaded with the metadata
        self.work_len = attn_work_len(m_cap, Hkv, max_blocks, max(1, self.workers))
        self.work = torch.zeros(self.work_len, dtype=torch.int32, device=device)

    def set_work(self, seq_lens_host):
        """Synchronous upload of the work list for ``seq_lens_host`` (tests /
        smoke; the engine stages it through its pinned metadata ring)."""
        w = attn_work_list(seq_lens_host, self.Hkv, self.workers)
        n = attn_work_used(w)
        self.work[:n].copy_(torch.from_numpy(w[:n]))


def attn_work_used(work) -> int:
    """Ints of a built work list that the kernel reads (the upload size)."""
    return (3 + int(work[0]) + 3) // 4 * 4 + 4 * int(work[1])


def attn_work_list(seq_lens, hkv: int, workers: int, out=None, maxp: int = ATTN_MAXP, minq: int = ATTN_MINQ):
    """The step's attention work list (mirrors pm_attn_work_list).  Units are
    the (row, kv head) pairs in row-major order, each nb = ceil(seq / 16)
    blocks; their blocks laid end to end (B in all) are cut into one range of
    q = max(minq, ceil(B / workers)) blocks per warp and every (unit x warp)
    segment into pieces of at most ``maxp`` blocks.  A piece is
    ``(row | kvh << 16, b0 | nblk << 16, chunk | nchunks << 16, seq)`` where
    chunk / nchunks are its rank / count among its unit's pieces (the merge
    order).  Layout: ``out[0]`` = warps used, ``out[1]`` = pieces P,
    ``out[2 : 3 + warps]`` = each warp's first piece (+ end), pieces from
    the next 16-byte boundary.  Every warp streams the same number of KV blocks
    (+-1 piece boundary), whatever the rows' lengths; the split points depend
    on the whole step, so attention results depend on the micro-batch's
    composition at fp32-rounding level (deterministic for a given step)."""
    import numpy as np
    seq = np.asarray(seq_lens, dtype=np.int64)
    nb = (seq + 15) // 16
    unb = np.repeat(nb, hkv)
    ustart = np.zeros(len(unb) + 1, dtype=np.int64)
    np.cumsum(unb, out=ustart[1:])
    B = int(ustart[-1])
    if B == 0 or workers <= 0:
        if out is None:
            out = np.zeros(3, dtype=np.int32)
        out[0] = out[1] = out[2] = 0
        return out
    q = max(minq, -(-B // workers))
    w_used = -(-B // q)
    wstart = np.minimum(np.arange(w_used + 1, dtype=np.int64) * q, B)
    cuts = np.union1d(ustart, wstart)
    seg_s, seg_e = cuts[:-1], cuts[1:]
    k = (seg_e - seg_s + maxp - 1) // maxp
    rep = np.repeat(np.arange(len(seg_s)), k)
    first = np.cumsum(k) - k
    ps = seg_s[rep] + (np.arange(int(k.sum())) - first[rep]) * maxp
    pe = np.minimum(ps + maxp, seg_e[rep])
    u = np.searchsorted(ustart, ps, side="right") - 1
    P = len(ps)
    chunk = np.arange(P) - np.searchsorted(u, u, side="left")
    nchunks = np.bincount(u, minlength=len(unb))[u]
    w = ps // q
    woff = np.searchsorted(w, np.arange(w_used + 1), side="left")
    r, h = u // hkv, u % hkv
    base = (3 + w_used + 3) // 4 * 4          # pieces 16-byte aligned (int4 loads)
    need = base + 4 * P
    if out is None:
        out = np.zeros(need, dtype=np.int32)
    assert len(out) >= need, "work list buffer too small"
    out[0], out[1] = w_used, P
    out[2:3 + w_used] = woff
    pc = out[base:base + 4 * P].reshape(P, 4)
    pc[:, 0] = r | (h << 16)
    pc[:, 1] = (ps - ustart[u]) | ((pe - ps) << 16)
    pc[:, 2] = chunk | (nchunks << 16)
    pc[:, 3] = seq[r]
    return out


def attn_workers(hd: int) -> int:
    """Warps of a full attention launch on this device (pm_attn_workers)."""
    return _C.lib().pm_attn_workers(hd)


# Launch configuration of the attention kernel (warps x KV-ring stages per SM;
# both keep 24 ring slots per SM).  With the balanced work split every warp
# streams the same number of blocks, so the choice is a measured rule on the
# step's rows (profiles/r2/attention_balanced.md).
ATTN_WIDE_ROWS = 96   # rows per step from which 12 warps x 2 stages beats 8 x 3


def choose_attn_cfg(rows: int, hkv: int, hd: int, max_blocks: int) -> int:
    """Launch configuration of a workspace's attention kernel: 12 warps x 2
    stages for wide steps (C2, ~121 rows: 5.66 vs 5.74 ms/step), 8 x 3 below
    (C3 stage, 48 rows: 1.925 vs 1.958; C4 stage equal) -- measured with the
    balanced split (profiles/r2/attention_balanced.md).  Never changes
    results beyond the split points (the work list is built for the chosen
    warp count); PM_ATTN_CFG forces one."""
    import os
    if os.environ.get("PM_ATTN_CFG"):
        return int(os.environ["PM_ATTN_CFG"])
    return 1 if rows >= ATTN_WIDE_ROWS else 2


ATTN_EARLY = _os.environ.get("PM_ATTN_EARLY", "1") == "1"   # A/B switch


def paged_attention(tmap_kv, q, block_table, seq_lens, out, ws: AttnWorkspace, M, H, Hkv, hd, layer,
                    L_s, stream=None, kv_tokens=0, decode=False):
    """``kv_tokens`` (sum of seq_lens, host-known) only feeds the optional timer.
    ``decode``: every row is a different request whose only new KV is its
    current token (not a prefill chunk), so the kernel may load the blocks
    before each row's last ahead of its dependency wait (cfg bit 5)."""
    cfg = ws.cfg if ws.cfg >= 0 else int(_os.environ.get("PM_ATTN_CFG", "1"))
    if isinstance(tmap_kv, PoolMap):
        cfg |= 16   # the map kind travels with the call (bit 4)
    if decode and ATTN_EARLY:
        cfg |= 32

    def go():
        _C.call("pm_paged_attention", tmap_kv.ptr, _ptr(q), _ptr(block_table), _ptr(seq_lens), _ptr(ws.work), _ptr(out),
                _ptr(ws.o), _ptr(ws.ml), _ptr(ws.counters), M, H, Hkv, hd, layer, L_s, block_table.shape[1],
                ws.max_chunks, ATTN_MAXP, cfg, _stream(stream))
    if TIMER is None:
        go()
    else:
        TIMER.around("attention", kv_tokens * 2 * Hkv * hd * 2 + 2 * M * H * hd * 2, stream, go)


def argmax_reduce(ws: GemmWorkspace, n_units, M, out_ids, tok_table=None, slots=None, stream=None):
    """Greedy ids from the lm_head GEMM's per-tile partials (``n_units`` =
    the lm_head's 256-row units; two 128-row argmax tiles each)."""
    _C.call("pm_argmax_reduce", _ptr(ws.amax_val), _ptr(ws.amax_idx), 2 * n_units, M, ws.m_cap, _ptr(out_ids),
            _ptr(tok_table), _ptr(slots), _stream(stream))
