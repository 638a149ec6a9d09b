"""Prefill with layer-wise asynchronous KV offload.

B200 counterpart of the reference's simulated prefill (REF = reference
``pkg/src/pipemax``): ``_prefill_run`` / ``simulate_prefill``
(pipeline_sim.py:241-323).  The reference pipelines each request through the
stages, streams every layer's KV to host memory as soon as that layer is
computed (``d2h.submit_stream`` per layer, :297-305) and bounds the staging
memory to ``staging_pool_requests`` requests whose offload has not drained
(:275-285, "offload_backpressure" stalls).

Here the same schedule runs on the real decode path:

* a prompt is processed in chunks of up to ``m_cap`` tokens with the decode
  kernels themselves -- every chunk row is a token at its own position, the
  fused QKV epilogue appends its K/V to the request's blocks and the paged
  attention kernel reads the request's KV up to that position (causal), so a
  later chunk attends to the earlier chunks straight from the pool;
* after layer ``l`` of a chunk the compute stream records an event and the
  stage's D2H copy stream moves that layer's new K/V (4 KB per token on
  Qwen3-8B, one pitched copy per run of physical blocks) into the request's
  block-first host replica, overlapping the next layers;
* requests that are resident for decode prefill straight into their own
  blocks; the others use free pool blocks as staging, at most
  ``staging_pool_requests`` of them in flight -- before a staging area is
  reused the compute stream waits for the D2H event of the request that last
  used it (the reference's backpressure stall, measured with CUDA events);
* the last prompt token's greedy id is the request's first generated token.

Times in the returned trace are CUDA-event times (seconds) since the start of
the prefill.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _C
from .model_core import blocks_for_tokens
from .trace import EventTrace


class _Clock:
    """CUDA-event timestamps relative to one origin event."""

    def __init__(self, stream):
        self.origin = torch.cuda.Event(enable_timing=True)
        self.origin.record(stream)
        self.pending = []   # (event, kind, payload)

    def mark(self, stream, kind, **payload):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        self.pending.append((ev, kind, payload))
        return ev

    def flush(self, trace: EventTrace):
        torch.cuda.synchronize()
        for ev, kind, payload in self.pending:
            trace.emit(self.origin.elapsed_time(ev) * 1e-3, kind, **payload)
        self.pending = []


def _runs(blocks):
    """Consecutive physical-block runs of a logical block list:
    [(first logical index, first physical id, length)]."""
    out = []
    for i, b in enumerate(blocks):
        if out and out[-1][1] + out[-1][2] == b:
            out[-1] = (out[-1][0], out[-1][1], out[-1][2] + 1)
        else:
            out.append((i, b, 1))
    return out


class PrefillRunner:
    """Runs the prefill phase of one episode on a ``DecodeEngine``'s stage
    executors, KV pools and host replicas."""

    def __init__(self, engine, staging_pool_requests: int = 2, offload: bool = True):
        if staging_pool_requests < 1:
            raise ValueError("staging_pool_requests must be >= 1")
        self.eng = engine
        self.staging = staging_pool_requests
        self.offload = offload
        self.d2h_bytes = 0
        self.stall_seconds = 0.0

    # ------------------------------------------------------------------ copies
    def _offload_layer(self, si, rid, table, p0, p1, li):
        """Layer ``li`` K/V of tokens [p0, p1) of ``rid``: pool -> replica,
        one pitched copy per run of consecutive physical blocks."""
        ex, kv = self.eng.stages[si]
        tb, bb = ex.tok_bytes, ex.block_bytes
        width = 2 * ex.spec.Hkv * ex.spec.hd * 2
        lay = li * width
        host0 = kv.rep.offset(self.eng.slot_of[rid])
        lb0, lb1 = p0 // 16, (p1 - 1) // 16
        for first, phys, n in _runs(table[lb0:lb1 + 1]):
            lb = lb0 + first
            t0 = max(p0, lb * 16)
            t1 = min(p1, (lb + n) * 16)
            src = kv.pool_ptr + phys * bb + (t0 - lb * 16) * tb + lay
            dst = kv.rep.ptr + host0 + t0 * tb + lay
            _C.call("pm_copy_2d", _C.C.c_void_p(dst), tb, _C.C.c_void_p(src), tb, width, t1 - t0,
                    _C.C.c_void_p(kv.d2h.cuda_stream))
            self.d2h_bytes += width * (t1 - t0)

    # ------------------------------------------------------------------ run
    def run(self, prompts: dict, order=None):
        """Prefill every request in ``order`` (default: ascending id).
        Returns (EventTrace, makespan_seconds)."""
        eng = self.eng
        ctl = eng.control
        trace = EventTrace()
        ex0, kv0 = eng.stages[0]
        exL = eng.stages[-1][0]
        clock = _Clock(kv0.compute)
        rids = list(order) if order is not None else sorted(prompts)
        resident = dict(ctl.alloc.tables)
        used = {b for t in resident.values() for b in t}
        free = [b for b in range(ctl.alloc.total) if b not in used]
        # staging areas for non-resident requests (each big enough for the
        # longest non-resident prompt), recycled round robin
        need = max([blocks_for_tokens(len(prompts[r]), 16) for r in rids if r not in resident] or [0])
        n_areas = min(self.staging, len(free) // need) if need else 0
        if need and n_areas < 1:
            raise RuntimeError(f"prefill staging needs {need} free blocks, pool has {len(free)}")
        areas = [free[i * need:(i + 1) * need] for i in range(n_areas)]
        area_done = [None] * n_areas      # per area: last request's D2H-done events (per stage)
        k_area = 0
        m_cap = eng.m_cap
        for rid in rids:
            prompt = np.asarray(prompts[rid], dtype=np.int64)
            L = len(prompt)
            if rid in resident:
                table = resident[rid]
                assert len(table) >= blocks_for_tokens(L, 16), f"request {rid}: table shorter than its prompt"
            else:
                a = k_area % n_areas
                k_area += 1
                table = areas[a][:blocks_for_tokens(L, 16)]
                if area_done[a] is not None:
                    # bounded staging: the area's previous request must have drained
                    for si, (ex, kv) in enumerate(eng.stages):
                        rdy = clock.mark(kv.compute, "stall_start", stage=si, request=int(rid),
                                         reason="offload_backpressure")
                        kv.compute.wait_event(area_done[a][si])
                        clock.mark(kv.compute, "stall_end", stage=si, request=int(rid),
                                   reason="offload_backpressure")
                        del rdy
            for p0 in range(0, L, m_cap):
                p1 = min(L, p0 + m_cap)
                n = p1 - p0
                last_chunk = p1 == L
                self._chunk(rid, table, prompt[p0:p1], p0, last_chunk, clock)
            if rid not in resident:
                evs = []
                for ex, kv in eng.stages:
                    ev = torch.cuda.Event()
                    ev.record(kv.d2h)
                    evs.append(ev)
                area_done[(k_area - 1) % n_areas] = evs
        # first generated tokens computed by the last stage -> stage 0's table
        if len(eng.stages) > 1:
            with torch.cuda.stream(kv0.compute):
                ex0.tok_table.copy_(exL.tok_table)
        for si, (ex, kv) in enumerate(eng.stages):
            clock.mark(kv.d2h, "offload_drained", stage=si)
        clock.flush(trace)
        trace.finalize()
        makespan = max((ev.time for ev in trace.events), default=0.0)
        self.stall_seconds = _paired(trace, "stall_start", "stall_end")
        return trace, makespan

    def _chunk(self, rid, table, tokens, p0, last_chunk, clock):
        """One prompt chunk through every stage, layer-wise offload hooks."""
        eng = self.eng
        n = len(tokens)
        M = eng.bucket(n)
        positions = list(range(p0, p0 + n))
        # metadata through the engine's ring: every row uses the request's
        # table; the last row of the last chunk sends its greedy id to the slot
        eng._upload_meta_rows(table, positions, M, last_slot=eng.slot_of[rid] if last_chunk else None)
        prev_ev = None
        for si, (ex, kv) in enumerate(eng.stages):
            s = kv.compute
            if prev_ev is not None:
                s.wait_event(prev_ev)
            with torch.cuda.stream(s):
                if ex.first:
                    ex.prefill_tokens[:n].copy_(torch.from_numpy(tokens.astype(np.int32)), non_blocking=True)
                    if M > n:
                        ex.prefill_tokens[n:M].fill_(0)
                if si > 0:
                    ex.resid[:M].copy_(eng.stages[si - 1][0].resid[:M])
                clock.mark(s, "stage_compute_start", phase="prefill", stage=si, request=int(rid), tokens=n)

                def hook(li, _si=si, _kv=kv):
                    if not self.offload:
                        return
                    ev = torch.cuda.Event()
                    ev.record(_kv.compute)
                    _kv.d2h.wait_event(ev)
                    clock.mark(_kv.d2h, "transfer_start", channel=f"d2h{_si}", stage=_si, request=int(rid),
                               layer=li, tag="kv_offload")
                    self._offload_layer(_si, rid, table, p0, p0 + n, li)
                    clock.mark(_kv.d2h, "transfer_end", channel=f"d2h{_si}", stage=_si, request=int(rid),
                               layer=li, tag="kv_offload")
                ex.forward(M, s, prefill_tokens=True, layer_hook=hook)
                clock.mark(s, "stage_compute_end", phase="prefill", stage=si, request=int(rid))
            prev_ev = torch.cuda.Event()
            prev_ev.record(s)
        if len(eng.stages) > 1:
            eng.stages[0][1].compute.wait_event(prev_ev)


def _paired(trace, a, b):
    starts = {}
    total = 0.0
    for ev in trace.events:
        key = (ev.payload.get("stage"), ev.payload.get("request"))
        if ev.kind == a:
            starts[key] = ev.time
        elif ev.kind == b and key in starts:
            total += ev.time - starts.pop(key)
    return total


def run_prefill(requests: dict, prompts: dict, cfg, params, spec, *, offload: bool = True,
                staging_pool_requests: int = 2, pp: int = 1, device="cuda", **kw):
    """``simulate_prefill``-shaped driver (REF pipeline_sim.py:308-323) on
    B200: prefill ``requests`` (id -> Request) with real kernels and
    layer-wise KV offload to each stage's host replica.  Returns
    (EventTrace, makespan_seconds, engine) -- the engine (its pools and host
    replicas filled) can go straight into decode."""
    from . import scheduler as sched
    from .engine import DecodeEngine
    if not requests:
        raise ValueError("requests must be nonempty")
    ids = sorted(requests)
    state = sched.SchedulerState(n=cfg.n, batches=[set() for _ in range(cfg.n)],
                                 lengths={r: requests[r].prefix_len for r in ids}, gpu_resident=set(),
                                 cpu_pool=set(ids))
    eng = DecodeEngine(spec, state, cfg, params, requests, pp=pp, device=device, kv_init="none", **kw)
    runner = PrefillRunner(eng, staging_pool_requests=staging_pool_requests, offload=offload)
    trace, makespan = runner.run(prompts, order=ids)
    return trace, makespan, eng
