"""The B200 decode engine: the reference's ``simulate_decode`` driver shape
over real hardware.

``run_decode(state, cfg, params, noise_spec, horizon, *, requests, ...)`` mirrors
``pipemax.pipeline_sim.simulate_decode`` (REF pkg/src/pipemax/
pipeline_sim.py:546-581) and returns ``(EventTrace, EpisodeMetrics)``; the
loop body is the reference's ``_DecodeEngine.run`` (:386-543) with the
simulated pieces replaced:

  reference                                  B200
  ---------                                  ----
  _plan_step / commit / GpuState counts      DecodeControl (same code path, run
                                             ahead of the GPU) + physical blocks
  estimate_decode_time x noise / n           StageExecutor.forward (sm_100a)
  h2d.submit_stream(kv_prefetch)             KvEngine.prefetch  (H2D copy stream)
  h2d.finish_stream -> stall                 compute-stream wait on the H2D event
  d2h.submit_stream(kv_offload_decode)       KvEngine.offload   (D2H copy stream)
  submit_high activation hop                 NCCL send/recv between stage ranks

With ``pp > 1`` in one process (``local_pipeline=True``) the stages run back
to back on one device -- used by tests to validate the layer split; the
multi-GPU path (one rank per stage) lives in ``pipeline.py``.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _C, ops
from .control import DecodeControl, StepWork
from .kv import HostReplica, KvEngine
from .model_core import ClusterConfig, EstimatorParams, blocks_for_tokens
from .models import ModelSpec, stage_layers
from .scheduler import SchedulerState
from .stage import StageExecutor
from .trace import EpisodeMetrics, EventTrace

# single-lane engines finish split-K units inside the GEMM kernels (one launch
# per projection) with PM_FUSED_FIXUP=1 -- measured slower than the post kernels
# (c3 stage 2.53 vs 1.94 ms/step, profiles/r2/fused_fixup.md), so opt-in
import os as _os
FUSED_FIXUP = _os.environ.get("PM_FUSED_FIXUP", "0") == "1"


class _MetaRing:
    """Mapped pinned host staging for per-step metadata (pm_host_alloc);
    ``depth`` buffers so the host can run ahead of the GPU without
    overwriting one a meta_upload kernel has not read yet."""

    def __init__(self, m_cap, max_blocks, depth=4, extra=0):
        import ctypes
        n = m_cap * (max_blocks + 3) + extra
        self.bufs, self.dev_ptrs, self._raw = [], [], []
        for _ in range(depth):
            p = _C.C.c_void_p()
            _C.call("pm_host_alloc", n * 4, _C.C.byref(p))
            d = _C.C.c_void_p()
            _C.call("pm_host_device_ptr", p, _C.C.byref(d))
            arr = (ctypes.c_int32 * n).from_address(p.value)
            self.bufs.append(torch.frombuffer(arr, dtype=torch.int32))
            self.dev_ptrs.append(d.value)
            self._raw.append(p.value)
        self.events = [None] * depth
        self.i = 0
        self.m_cap, self.max_blocks = m_cap, max_blocks

    def next(self):
        k = self.i % len(self.bufs)
        self.i += 1
        for ev in self.events[k] or ():
            ev.synchronize()
        return k, self.bufs[k]

    def __del__(self):
        try:
            for p in self._raw:
                _C.call("pm_host_free", _C.C.c_void_p(p))
        except Exception:
            pass


def attn_rows_hint(n_requests: int, micro_batches: int) -> int:
    """Rows of a typical rotation step: one micro-batch of the requests."""
    return -(-n_requests // max(1, micro_batches))


class DecodeEngine:
    def __init__(self, spec: ModelSpec, state: SchedulerState, cfg: ClusterConfig, params: EstimatorParams,
                 requests: dict, *, pp: int = 1, device="cuda", mode="dynamic", quota_tokens=0,
                 seed: int = 0, m_cap: int = None, timing=True, kv_init="random", prompts=None,
                 record_logits=False, max_pos=None, trace: EventTrace = None, graphs: bool = True,
                 local_stages=None, staging_pool_requests: int = 2, lanes: int = None,
                 copy_priority: bool = True, calibrate: bool = False):
        """``local_stages``: which of the ``pp`` stages this process hosts
        (default all; one rank per stage under torchrun, see pipeline.py)."""
        self.spec, self.cfg, self.params = spec, cfg, params
        self.staging_pool_requests = staging_pool_requests
        self.requests = requests
        self.dev = torch.device(device)
        self.metrics = EpisodeMetrics()
        self.trace = trace if trace is not None else EventTrace()
        self.control = DecodeControl(state, cfg, params, requests, mode=mode, quota_tokens=quota_tokens,
                                     metrics=self.metrics)
        bs = cfg.block_size
        assert bs == 16, "the kernels use 16-token blocks"
        rids = sorted(requests)
        self.slot_of = {rid: i for i, rid in enumerate(rids)}
        max_len = max(r.input_len + r.output_len for r in requests.values())
        self.max_blocks = blocks_for_tokens(max_len + 1, bs)
        self.m_cap = m_cap or len(rids)
        self.max_pos = max_pos or (self.max_blocks * bs)
        # +1 physical block and +1 token slot: padding rows of a bucketed
        # micro-batch point there, so CUDA graphs are captured per 16-row bucket
        pool_blocks = self.control.alloc.total + 1
        self.trash_block = self.control.alloc.total
        self.trash_slot = len(rids)
        self.graphs = graphs
        self.stages = []
        self.pp = pp
        if lanes is None:
            lanes = 2 if (pp == 1 and local_stages is None) else 1
            if _os.environ.get("PM_LANES"):   # A/B and debugging
                lanes = int(_os.environ["PM_LANES"])
        for s in (range(pp) if local_stages is None else local_stages):
            ex = StageExecutor(spec, stage_layers(spec, pp, s), first=(s == 0), last=(s == pp - 1),
                               m_cap=self.m_cap, pool_blocks=pool_blocks, max_blocks=self.max_blocks,
                               n_slots=len(rids) + 1, device=self.dev, seed=seed, max_pos=self.max_pos,
                               keep_logical=record_logits,
                               gemm_sms=ops.GEMM_CTAS_1LANE if lanes == 1 else None,
                               rows_hint=attn_rows_hint(self.m_cap, cfg.n))
            if record_logits:
                ex.enable_logits()
            rep = HostReplica(len(rids), self.max_blocks, ex.block_bytes, device=self.dev)
            self.stages.append((ex, KvEngine(ex, rep, self.slot_of, self.dev, timing=timing,
                                             low_priority_copies=copy_priority)))
        self.work_len = self.stages[0][0].aws.work_len
        self.attn_hkv, self.attn_workers = self.stages[0][0].aws.Hkv, self.stages[0][0].aws.workers
        self.meta = _MetaRing(self.m_cap, self.max_blocks, extra=self.work_len)
        # lanes = micro-batches in flight on one GPU: consecutive rotation steps
        # (different micro-batches, independent compute) run on their own
        # compute streams with their own activation buffers and graphs, so one
        # step's latency-bound kernels overlap the other's weight streaming.
        # Ordering through the KV pool stays event-based per step (KvEngine).
        self.serialize_lanes = False   # True: step t waits for step t-1 (per-kernel timing passes)
        self.lanes = lanes
        # one micro-batch in flight: nothing overlaps the fused norm's arrival
        # chain, and fixup + a row-parallel norm kernel measured faster
        split = lanes == 1
        if _os.environ.get("PM_SPLIT_NORM"):   # A/B
            split = _os.environ["PM_SPLIT_NORM"] == "1"
        for ex, _ in self.stages:
            ex.split_norm = split
            if lanes == 1 and FUSED_FIXUP:
                ex.enable_fused()
        self.lane_stages = [self.stages]
        for li in range(1, lanes):
            self.lane_stages.append([(ex.clone_lane(), kv) for ex, kv in self.stages])
            for _, kv in self.stages:
                assert kv.add_lane() == li
        self.record_logits = record_logits
        self.logits_log = []   # (t, rows, positions, logits[M, V]) when recording (np, or torch if "device")
        self.ids_log = []      # (t, rows, ids np)
        self.t = 0
        self.n_evicted = self.n_prefetched = 0
        if graphs:  # one graph per 16-row bucket and lane, captured up front
            for li, stages in enumerate(self.lane_stages):
                for ex, kv in stages:
                    for Mb in range(16, self.m_cap + 16, 16):
                        ex.capture(min(Mb, self.m_cap), kv.streams[li])
        self.calibration = None
        if calibrate:
            # on-box estimator fit (REF model_core.py:158-182) BEFORE the KV is
            # seeded (the profile appends KV at synthetic positions), then the
            # planner plans with it: T_hat -> the prefetch budget B * T_hat
            self.recalibrate()
        self._init_kv(kv_init, prompts, seed)

    # ------------------------------------------------------------------ setup
    def _init_kv(self, how, prompts, seed):
        """Seed every request's KV: the host replica holds all of it, the
        resident requests' blocks also sit in HBM (REF run_episode's initial
        bulk load, pipeline_sim.py:732-739)."""
        rids = sorted(self.requests)
        g = torch.Generator(device=self.dev).manual_seed(seed + 1)
        first_tok = torch.randint(0, self.spec.vocab, (len(rids) + 1,), generator=g, device=self.dev,
                                  dtype=torch.int32)
        # every stage's table starts equal: with several local stages the last
        # stage's table is copied back to stage 0's after each step (the
        # last -> first hop), so it must hold the not-yet-executed rows' tokens too
        for ex, kv in self.stages:
            ex.tok_table.copy_(first_tok)
        torch.cuda.synchronize()
        if how == "prefill":
            assert prompts is not None
            self._prefill(prompts)
            return
        if how == "none":   # caller fills the KV (prefill.run_prefill)
            return
        # timing runs: random KV in HBM for resident blocks and in the host
        # replica for the others (seeded: the replica's pinned pages may be
        # recycled host memory, and two processes must hold the same values)
        for ex, kv in self.stages:
            # seeded per stage (its first layer), so a rank hosting one stage of a
            # pipeline holds the same KV as a process hosting all of them
            gs = torch.Generator(device=self.dev).manual_seed(seed + 1 + 1000 * (ex.layers[0] + 1))
            pv = ex.pool.view(ex.pool_blocks, -1)
            for rid, blocks in self.control.alloc.tables.items():
                idx = torch.tensor(blocks, device=self.dev)
                pv[idx] = (torch.randn(len(blocks), pv.shape[1], generator=gs, device=self.dev) * 0.5).to(torch.bfloat16)
            bb = kv.block_bytes
            for rid in rids:
                if rid in self.control.alloc.tables:
                    continue
                nb = min(-(-self.requests[rid].prefix_len // 16), kv.rep.max_blocks)
                if nb <= 0:
                    continue
                buf = (torch.randn(nb, bb // 2, generator=gs, device=self.dev) * 0.5).to(torch.bfloat16)
                base = kv.rep.offset(self.slot_of[rid])
                d = np.arange(nb, dtype=np.int64) * bb + base
                s = np.arange(nb, dtype=np.int64) * bb
                _C.call("pm_copy_pieces", _C.C.c_void_p(kv.rep.ptr), _C.C.c_void_p(buf.data_ptr()),
                        d.ctypes.data_as(_C.C.c_void_p), s.ctypes.data_as(_C.C.c_void_p), nb, bb,
                        _C.C.c_void_p(torch.cuda.current_stream().cuda_stream))
                torch.cuda.current_stream().synchronize()
        torch.cuda.synchronize()

    def _prefill(self, prompts):
        """Real prefill of every request (chunked, layer-wise async KV offload
        to the host replicas, bounded staging -- prefill.PrefillRunner, REF
        pipeline_sim.py:241-323).  Resident requests end with their KV in
        their own blocks and on the host; the others on the host only."""
        from .prefill import PrefillRunner
        self.prefill_runner = PrefillRunner(self, staging_pool_requests=self.staging_pool_requests)
        self.prefill_trace, self.prefill_makespan = self.prefill_runner.run(prompts)

    # ------------------------------------------------------------------ per step
    def bucket(self, M):
        return min(self.m_cap, -(-M // 16) * 16) if self.graphs else M

    def _upload_meta(self, rows, positions, tables, stream=None, lane=0):
        """Block tables, positions, seq lens and slots of the step's rows,
        padded to the 16-row bucket with rows aimed at the trash block/slot.
        Returns the physical blocks the step reads / writes (the KV engine's
        block-hazard record: a later prefetch into one of them must wait for
        this step's compute)."""
        self._fill_meta([tables[r] for r in rows], positions, [self.slot_of[r] for r in rows], stream, lane)
        return self._last_used_blocks

    def _upload_meta_rows(self, table, positions, M=None, last_slot=None, stream=None):
        """Prefill chunk: every row is a token of one request (its block
        table); greedy ids go to the trash slot except the last row's, which
        goes to ``last_slot`` when given (the request's first generated token)."""
        n = len(positions)
        slots = [self.trash_slot] * n
        if last_slot is not None:
            slots[-1] = last_slot
        self._fill_meta([table] * n, positions, slots, stream)

    def _fill_meta(self, row_tables, positions, slots, stream=None, lane=0):
        n, mb = len(row_tables), self.max_blocks
        M = self.bucket(n)
        k, buf = self.meta.next()
        a = buf.numpy()
        bt = a[:M * mb].reshape(M, mb)
        bt[:] = 0
        for i, tb in enumerate(row_tables):
            bt[i, :len(tb)] = tb
        # physical blocks the step reads/writes (rows' blocks up to their position)
        nb = np.asarray(positions, dtype=np.int64) // 16 + 1
        self._last_used_blocks = bt[:n][np.arange(mb)[None, :] < nb[:, None]].astype(np.int64)
        bt[n:, 0] = self.trash_block
        o = M * mb
        a[o:o + n] = positions
        a[o + n:o + M] = 0
        a[o + M:o + M + n] = np.asarray(positions) + 1
        a[o + M + n:o + 2 * M] = 1
        a[o + 2 * M:o + 2 * M + n] = slots
        a[o + 2 * M + n:o + 3 * M] = self.trash_slot
        # balanced attention work list over the bucket's rows, padding rows included
        wo = o + 3 * M
        ops.attn_work_list(a[o + M:o + 2 * M], self.attn_hkv, self.attn_workers, a[wo:wo + self.work_len])
        wn = ops.attn_work_used(a[wo:])
        evs = []
        base = self.meta.dev_ptrs[k]
        srcs = (_C.C.c_void_p * 5)(base, base + 4 * o, base + 4 * (o + M), base + 4 * (o + 2 * M), base + 4 * wo)
        counts = (_C.C.c_int * 5)(M * mb, M, M, M, wn)
        for ex, kv in self.lane_stages[lane]:
            s = kv.streams[lane] if stream is None else stream
            dsts = (_C.C.c_void_p * 5)(ex.block_table.data_ptr(), ex.positions.data_ptr(), ex.seq_lens.data_ptr(),
                                       ex.slots.data_ptr(), ex.aws.work.data_ptr())
            _C.call("pm_meta_upload", 5, dsts, srcs, counts, _C.C.c_void_p(s.cuda_stream))
            ev = torch.cuda.Event()
            ev.record(s)
            evs.append(ev)
        self.meta.events[k] = evs

    def _forward_all(self, n, kv_tokens=0, lane=0):
        """Run the stages in order on the lane's compute streams (single
        process: stage s+1 waits for stage s's activations via an event)."""
        M = self.bucket(n)
        stages = self.lane_stages[lane]
        prev_ev = None
        for si, (ex, kv) in enumerate(stages):
            st = kv.streams[lane]
            if si > 0:
                # the inter-stage hop as the multi-GPU pipeline sends it: the
                # previous stage packs its residual to bf16, this stage unpacks
                prev = stages[si - 1][0]
                hop = self._hop_buffer(lane, prev.resid)
                n_el = M * prev.resid.shape[1]
                _C.call("pm_hop_pack", _C.C.c_void_p(prev.resid.data_ptr()), _C.C.c_void_p(hop.data_ptr()), n_el,
                        _C.C.c_void_p(stages[si - 1][1].streams[lane].cuda_stream))
                prev_ev = torch.cuda.Event()
                prev_ev.record(stages[si - 1][1].streams[lane])
                st.wait_event(prev_ev)
                _C.call("pm_hop_unpack", _C.C.c_void_p(hop.data_ptr()), _C.C.c_void_p(ex.resid.data_ptr()), n_el,
                        _C.C.c_void_p(st.cuda_stream))
            with torch.cuda.stream(st):
                ex.run(M, st, graphs=self.graphs, kv_tokens=kv_tokens)
                if si == len(stages) - 1 and len(stages) > 1:
                    # greedy ids back to stage 0's token table (the last->first hop)
                    stages[0][0].tok_table.copy_(ex.tok_table)
            prev_ev = torch.cuda.Event()
            prev_ev.record(st)
        if len(stages) > 1:
            stages[0][1].streams[lane].wait_event(prev_ev)

    def recalibrate(self, grid=None, reps: int = 3):
        """Fit (alpha, beta, delta) to this engine's measured step periods (its
        lane mode included) and plan every later step with the fit."""
        from .calibrate import calibrate_on_device, default_grid
        if grid is None:   # batch sizes around a micro-batch's rows, lengths up to the longest request
            grid = default_grid(min(self.m_cap, 2 * attn_rows_hint(self.m_cap, self.cfg.n)), self.max_blocks * 16 - 1)
        params, samples, err = calibrate_on_device(self, grid, reps)
        self.params = params
        self.control.params = params
        self.calibration = {"params": params, "samples": samples, "max_rel_fit_err": err}
        torch.cuda.synchronize()
        return params

    def refit_online(self, skip: int = 1):
        """Closed loop on the running engine: the planner's predicted step time
        vs the measured step period of the steps run so far (CUDA events, this
        engine's lane mode and transfer load included) -> shift delta by the
        median error, so the prefetch budget B * T_hat follows the box.  alpha and
        beta keep the on-box grid fit (the running steps span too little of
        (b, L) to refit them).  Returns the shift in seconds."""
        from .calibrate import step_errors
        torch.cuda.synchronize()
        pairs = step_errors(self.stages[0][1].records)[skip:]
        if self.lanes > 1:
            # two micro-batches in flight: the period is the overlapped interval,
            # not a step's time, and planning with the shifted delta measured
            # 10 % slower at C2 (profiles/r2/ab/refit.md) -- keep the grid fit
            self.refit = {"shift_s": 0.0, "periods": len(pairs), "skipped": "lanes > 1"}
            return 0.0
        if len(pairs) < 3:   # (the bench's 6 warm-up steps give 5 periods, 4 after the first)
            self.refit = {"shift_s": 0.0, "periods": len(pairs)}
            return 0.0
        shift = float(np.median([meas - pred for pred, meas in pairs]))
        p = self.params
        self.params = EstimatorParams(p.alpha, p.beta, max(p.delta + shift, 1e-6))
        self.control.params = self.params
        self.refit = {"shift_s": shift, "periods": len(pairs)}
        return shift

    def _hop_buffer(self, lane, resid):
        """bf16 wire buffer of the single-process stage hop (one per lane)."""
        if not hasattr(self, "_hops"):
            self._hops = {}
        b = self._hops.get(lane)
        if b is None:
            b = self._hops[lane] = torch.empty(resid.numel(), dtype=torch.bfloat16, device=resid.device)
        return b

    def start_phase(self, control: DecodeControl):
        """Begin a new decode phase with ``control`` (episode.py): the
        weights, KV pool, host replicas, token table, lanes and graphs stay;
        the resident requests' KV is loaded from their host replicas into the
        blocks the new control plane assigned."""
        torch.cuda.synchronize()
        self.control = control
        self.t = 0
        for ex, kv in self.stages:
            kv.reset_phase()
            kv.load_resident(control.alloc.tables)
        torch.cuda.synchronize()

    # ------------------------------------------------------------------ lanes
    def lane_of(self, t: int) -> int:
        return t % self.lanes

    def last_executor(self, t: int):
        """The last stage's executor that ran step ``t`` (its out_ids/logits)."""
        return self.lane_stages[self.lane_of(t)][-1][0]

    def begin_region(self, ev):
        """Record ``ev`` on lane 0's first-stage stream; every other lane's
        streams wait for it (start of a timed region)."""
        ev.record(self.stages[0][1].streams[0])
        for ex, kv in self.stages:
            for st in kv.streams:
                st.wait_event(ev)

    def end_region(self, ev):
        """Record ``ev`` after all work of every lane (end of a timed region)."""
        s0 = self.stages[0][1].streams[0]
        for ex, kv in self.stages:
            for st in kv.streams:
                if st is not s0:
                    e = torch.cuda.Event()
                    e.record(st)
                    s0.wait_event(e)
        ev.record(s0)

    def step(self) -> StepWork:
        work = self.control.step()
        if work is None:
            return None
        t = self.t
        M = len(work.rows)
        self.n_evicted += len(work.evicted) + len(work.relief_evicted)
        self.n_prefetched += len(work.prefetch)
        lane = self.lane_of(t)
        stages = self.lane_stages[lane]
        recs = []
        info = {"plan": work.plan, "batch_tokens": work.batch_tokens, "completed": list(work.completed),
                "resident_tokens": self.control.resident_tokens, "capacity_tokens": self.control.capacity_tokens}
        for ex, kv in stages:
            rec = {"t": t, "M": M, "info": info, "stream": kv.streams[lane], "lane": lane,
                   "serialize": self.serialize_lanes}
            kv.prefetch(t, work, rec)
            recs.append(rec)
        self._upload_meta(work.rows, work.positions, work.tables, lane=lane)
        for (ex, kv), rec in zip(stages, recs):
            rec["used_blocks"] = self._last_used_blocks
            kv.before_compute(t, work, rec)
        self._forward_all(M, kv_tokens=sum(work.positions) + M, lane=lane)
        for (ex, kv), rec in zip(stages, recs):
            kv.after_compute(t, rec)
            kv.offload(t, work, rec)
        if self.record_logits and M:
            last = stages[-1][0]
            torch.cuda.synchronize()
            if self.record_logits == "device":   # keep on the GPU (real-shape parity tests)
                self.logits_log.append((t, list(work.rows), list(work.positions), last.logits[:M].clone()))
            else:
                self.logits_log.append((t, list(work.rows), list(work.positions), last.logits[:M].cpu().numpy()))
            self.ids_log.append((t, list(work.rows), last.out_ids[:M].cpu().numpy().copy()))
        self.t += 1
        return work

    def run(self, horizon=None):
        n = 0
        while horizon is None or n < horizon:
            if self.step() is None:
                break
            n += 1
        torch.cuda.synchronize()
        return n

    def emit_trace(self, origin, trace: EventTrace = None) -> EventTrace:
        """Decode events of every step so far in the reference's trace schema
        (REF pipeline_sim.py:410-421, 460-482, 505-510, 221-233), timed by the
        CUDA events the KV engines recorded, in seconds since ``origin``."""
        tr = trace if trace is not None else self.trace
        torch.cuda.synchronize()

        def ts(ev):
            return origin.elapsed_time(ev) * 1e-3

        for si, (ex, kv) in enumerate(self.stages):
            h2d_name, d2h_name = f"h2d{si}", f"d2h{si}"
            for rec in kv.records:
                if "start" not in rec or "end" not in rec:
                    continue
                info, p = rec.get("info", {}), rec.get("info", {}).get("plan")
                it, b = rec["t"], (p.exec_batch_index if p is not None else None)
                t0, t1 = ts(rec["start"]), ts(rec["end"])
                if "ready" in rec and t0 - ts(rec["ready"]) > 1e-6:
                    tr.emit(ts(rec["ready"]), "stall_start", iter=it, batch=b, stage=si, reason="prefetch_wait")
                    tr.emit(t0, "stall_end", iter=it, batch=b, stage=si, reason="prefetch_wait")
                payload = dict(phase="decode", stage=si, iter=it, batch=b)
                if si == 0 and p is not None:
                    payload.update(exec_seconds=t1 - t0, predicted_seconds=p.predicted_exec_seconds,
                                   batch_tokens=info["batch_tokens"], resident_tokens_total=info["resident_tokens"],
                                   next_residual_tokens=p.residual_tokens, next_prefetched_tokens=p.prefetch_tokens,
                                   budget_tokens=p.prefetch_budget_tokens, capacity_tokens=info["capacity_tokens"],
                                   steady=p.steady)
                tr.emit(t0, "stage_compute_start", **payload)
                tr.emit(t1, "stage_compute_end", phase="decode", stage=si, iter=it, batch=b)
                for kind, ch, direction, tag in (("h2d", h2d_name, "h2d", "kv_prefetch"),
                                                 ("d2h", d2h_name, "d2h", "kv_offload_decode")):
                    if f"{kind}_start" in rec:
                        pl = dict(channel=ch, direction=direction, priority="low", bytes=rec.get(f"{kind}_bytes", 0),
                                  tag=[tag, it])
                        tr.emit(ts(rec[f"{kind}_start"]), "transfer_start", **pl)
                        tr.emit(ts(rec[f"{kind}_end"]), "transfer_end", **pl)
                if si == len(self.stages) - 1:
                    for rid in info.get("completed", []):
                        tr.emit(t1, "request_complete", request=int(rid), iter=it)
        return tr

    def finalize_metrics(self, wall_seconds: float):
        m = self.metrics
        stall = h2d = d2h = 0.0
        for ex, kv in self.stages:
            s, a, b, _ = kv.timings()
            stall, h2d, d2h = max(stall, s), max(h2d, a), max(d2h, b)
        m.stall_seconds = stall
        m.h2d_busy_seconds, m.d2h_busy_seconds = h2d, d2h
        m.h2d_bytes = sum(kv.h2d_bytes for _, kv in self.stages)
        m.d2h_bytes = sum(kv.d2h_bytes for _, kv in self.stages)
        m.wall_seconds = m.decode_seconds = wall_seconds
        return m.finalize()


def _default_model(cfg: ClusterConfig) -> ModelSpec:
    """The model a reference-style call (no ``model=``) runs: the BASELINE
    shape whose whole-model KV bytes/token equals ``cfg.kv_bytes_per_token``,
    else the tiny C1 model (the planner's arithmetic -- capacity_blocks,
    budgets -- always comes from ``cfg`` itself)."""
    from .models import SPECS, TINY
    for spec in SPECS.values():
        if spec.kv_bytes_per_token() == cfg.kv_bytes_per_token:
            return spec
    return TINY


def run_decode(state: SchedulerState, cfg: ClusterConfig, params: EstimatorParams, noise_spec=None,
               horizon: int = None, *, requests: dict, seed: int = 0, actual_params=None,
               priority_enabled: bool = True, model=None, pp: int = 1, device="cuda", kv_init="random",
               prompts=None, **kw):
    """Drop-in for ``simulate_decode`` (REF pipeline_sim.py:546-549): the same
    positional order ``(state, cfg, params, noise_spec, horizon)`` and
    keywords ``requests, seed, actual_params, priority_enabled``; returns
    ``(EventTrace, EpisodeMetrics)``.

    * ``noise_spec`` / ``actual_params`` shape the reference's SIMULATED stage
      duration (``estimate_decode_time(actual_params) x noise``, REF :423-427);
      here durations are measured on the GPU, so both are accepted and unused.
    * ``priority_enabled`` (REF ChannelSim two-lane priority, transfer.py:
      195-213): True puts the KV copy streams at low stream priority under the
      compute streams; False gives them default priority (the orchestration-
      free baseline).
    * B200 extras (keyword-only): ``model`` -- a ModelSpec or name (default
      ``_default_model(cfg)``), ``pp`` stages in this process, ``kv_init``
      ("random" | "prefill" with ``prompts``), and DecodeEngine options.
    Raises ``ConfigError`` for a non-ClusterConfig ``cfg`` (REF :551-552)."""
    from .models import SPECS
    from .trace import ConfigError
    if not isinstance(cfg, ClusterConfig):
        raise ConfigError("cfg must be a ClusterConfig")
    if model is None:
        spec = _default_model(cfg)
    elif isinstance(model, str):
        if model not in SPECS:
            raise ConfigError(f"unknown model {model!r} (one of {sorted(SPECS)})")
        spec = SPECS[model]
    elif isinstance(model, ModelSpec):
        spec = model
    else:
        raise ConfigError(f"model must be a ModelSpec or a name, not {type(model).__name__}")
    eng = DecodeEngine(spec, state, cfg, params, requests, pp=pp, device=device, seed=seed,
                       kv_init=kv_init, prompts=prompts, copy_priority=priority_enabled, **kw)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    eng.run(horizon)
    end.record()
    torch.cuda.synchronize()
    wall = start.elapsed_time(end) * 1e-3
    m = eng.finalize_metrics(wall)
    eng.emit_trace(start)
    eng.trace.finalize()
    return eng.trace, m
