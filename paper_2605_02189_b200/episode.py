"""Episode-level prefill <-> decode switching.

The reference's ``run_episode`` (REF = reference ``pkg/src/pipemax``,
pipeline_sim.py:604-780) alternates two phases until the workload finishes:

* prefill: admit pending requests (ascending id) while the projected host KV
  stays under ``rho_hi * cpu_kv_capacity`` (the first one always, unless it
  exceeds the capacity), prefill them with layer-wise offload;
* decode: start from the prefill remnants (the last ``min(2n, #ready)`` ready
  requests resident, the rest in the host pool; ``policy="no_prefetch"``
  instead fills a closed, balanced resident set with each request's full
  growth reserved), bulk-load their KV, and decode until everything live fits
  on the GPUs again while the next pending prompt fits in host memory (or the
  horizon / the workload ends); survivors drop their GPU copies.

``run_episode`` reproduces that loop -- every admission, residency and
stop decision -- on top of ``DecodeControl`` (the engine's bit-exact control
plane).  ``ControlBackend`` runs the decisions alone (what
tests/test_episode_golden.py checks against the reference's own plan
stream); ``B200Backend`` executes them on the GPU: the real prefill with
layer-wise offload (prefill.PrefillRunner) and the decode engine, whose
weights, KV pool and host replicas persist across phases.
"""

from __future__ import annotations

from collections import deque

import numpy as np

from . import scheduler as sched
from .control import DecodeControl
from .model_core import (ClusterConfig, Request, blocks_for_tokens, capacity_blocks, per_batch_token_budget,
                         system_token_capacity)
from .trace import CapacityError, ConfigError, EpisodeMetrics, EventTrace


def parse_policy(policy):
    """(mode, static ratio) of a policy name (REF pipeline_sim.py:585-601)."""
    if policy == "dynamic":
        return "dynamic", None
    if policy in ("no_prefetch", "no_prefetch_pp"):
        return "none", None
    if isinstance(policy, tuple) and policy[0] == "static":
        ratio = float(policy[1])
    elif isinstance(policy, str) and policy.startswith("static:"):
        ratio = float(policy.split(":", 1)[1])
    else:
        raise ValueError(f"unknown policy {policy!r}")
    if not 0 < ratio <= 1:
        raise ValueError("static prefetch ratio must be in (0, 1]")
    return "static", ratio


class ControlBackend:
    """Decisions only: prefill is instantaneous, decode runs DecodeControl."""

    def __init__(self):
        self.phases = []

    def prefill(self, rids):
        self.phases.append(("prefill", list(rids)))
        return 0.0, 0.0

    def decode_phase(self, state, cfg, params, requests, metrics, mode, quota):
        self.phases.append(("decode", sorted(state.gpu_resident), sorted(state.cpu_pool)))
        return DecodeControl(state, cfg, params, requests, mode=mode, quota_tokens=quota, metrics=metrics)

    def step(self, ctl):
        return ctl.step()

    def end_decode_phase(self, ctl):
        return 0.0


class B200Backend(ControlBackend):
    """Runs the phases on the GPU through one DecodeEngine whose weights,
    pool and host replicas live for the whole episode."""

    def __init__(self, spec, cfg, params, requests, prompts, *, staging_pool_requests=2, seed=0, **engine_kw):
        super().__init__()
        import torch
        from .engine import DecodeEngine
        self.torch = torch
        ids = sorted(requests)
        boot = sched.SchedulerState(n=cfg.n, batches=[set() for _ in range(cfg.n)],
                                    lengths={r: requests[r].prefix_len for r in ids}, gpu_resident=set(),
                                    cpu_pool=set(ids))
        self.eng = DecodeEngine(spec, boot, cfg, params, requests, kv_init="none", seed=seed,
                                staging_pool_requests=staging_pool_requests, **engine_kw)
        self.requests = requests          # the episode advances these (the engine's own objects)
        self.prompts = prompts
        self.staging = staging_pool_requests
        self.tokens = 0
        self.decode_device_seconds = 0.0

    def prefill(self, rids):
        from .prefill import PrefillRunner
        super().prefill(rids)
        self.eng.control.alloc.tables.clear()       # survivors dropped their GPU copies
        runner = PrefillRunner(self.eng, staging_pool_requests=self.staging)
        trace, makespan = runner.run({r: self.prompts[r] for r in rids}, order=list(rids))
        return makespan, runner.stall_seconds

    def decode_phase(self, state, cfg, params, requests, metrics, mode, quota):
        super().decode_phase(state, cfg, params, requests, metrics, mode, quota)
        ctl = DecodeControl(state, cfg, params, requests, mode=mode, quota_tokens=quota, metrics=metrics)
        self.eng.start_phase(ctl)
        self._t0 = self.torch.cuda.Event(enable_timing=True)
        self.eng.begin_region(self._t0)
        return ctl

    def step(self, ctl):
        work = self.eng.step()
        if work is not None:
            self.tokens += len(work.rows)
        return work

    def end_decode_phase(self, ctl):
        t1 = self.torch.cuda.Event(enable_timing=True)
        self.eng.end_region(t1)
        self.torch.cuda.synchronize()
        sec = self._t0.elapsed_time(t1) * 1e-3
        self.decode_device_seconds += sec
        return sec


def run_episode(workload, cfg: ClusterConfig, params, policy="dynamic", seed: int = 0, *, backend=None,
                scheduler_knobs: dict = None, rho_hi: float = 0.9, horizon: int = None,
                trace: EventTrace = None) -> EpisodeMetrics:
    """The reference's episode loop (REF pipeline_sim.py:604-780) over
    ``backend`` (default: ``ControlBackend``).  ``workload`` is a list of
    Requests; their ``generated`` counts are advanced in place."""
    if not workload:
        raise ValueError("workload must be nonempty")
    if not isinstance(cfg, ClusterConfig):
        raise ConfigError("cfg must be a ClusterConfig")
    mode, ratio = parse_policy(policy)
    quota = int(ratio * system_token_capacity(cfg)) if ratio else 0
    for r in workload:
        if (r.input_len + r.output_len) * cfg.kv_bytes_per_token > cfg.cpu_kv_capacity:
            raise CapacityError(f"request {r.id} exceeds CPU KV capacity")
    knobs = dict(scheduler_knobs or {})
    if "ema_alpha" not in knobs:
        knobs["ema_alpha"] = 0.3
    backend = backend or ControlBackend()
    own_trace = trace if trace is not None else EventTrace()
    metrics = EpisodeMetrics()
    requests = getattr(backend, "requests", None) or {r.id: Request(r.id, r.input_len, r.output_len, r.generated)
                                                     for r in workload}
    pending = deque(sorted(requests.values(), key=lambda r: r.id))
    ready = []
    live_tokens = 0
    clock = 0.0
    cap_tokens = system_token_capacity(cfg)
    budget = per_batch_token_budget(cfg)
    cap_blocks = capacity_blocks(cfg)

    while pending or ready:
        # ------------------------------------------------ prefill phase
        admitted = []
        if pending:
            watermark = rho_hi * cfg.cpu_kv_capacity
            while pending:
                nxt = pending[0]
                projected = (live_tokens + nxt.input_len) * cfg.kv_bytes_per_token
                if admitted and projected > watermark:
                    break
                if projected > cfg.cpu_kv_capacity:
                    break
                pending.popleft()
                admitted.append(nxt)
                live_tokens += nxt.input_len
            if admitted:
                own_trace.emit(clock, "phase_switch", to="prefill", live_kv_tokens=live_tokens)
                metrics.phase_switches += 1
                sec, exposed = backend.prefill([r.id for r in admitted])
                metrics.prefill_seconds += sec
                metrics.exposed_offload_seconds += exposed
                clock += sec
                ready.extend(r.id for r in admitted)
        if not ready:
            break

        # ------------------------------------------------ decode phase
        own_trace.emit(clock, "phase_switch", to="decode", live_kv_tokens=live_tokens)
        metrics.phase_switches += 1
        assignment = {}
        if mode == "none":
            used_blocks = 0
            resident_ids = []
            totals = [0] * cfg.n
            for rid in ready:
                req = requests[rid]
                peak = req.prefix_len + (req.output_len - req.generated)
                blocks = blocks_for_tokens(peak, cfg.block_size)
                target = min(range(cfg.n), key=lambda idx: (totals[idx], idx))
                if totals[target] + peak > budget or used_blocks + blocks > cap_blocks:
                    break
                totals[target] += peak
                used_blocks += blocks
                assignment[rid] = target
                resident_ids.append(rid)
            if not resident_ids:
                break  # head request can never fit; stop rather than spin
        else:
            remnants = min(2 * cfg.n, len(ready))
            resident_ids = ready[-remnants:] if remnants else []
        resident_set = set(resident_ids)
        pool_ids = [rid for rid in ready if rid not in resident_set]
        lengths = {rid: requests[rid].prefix_len for rid in ready}
        if mode == "none":
            batches = [set() for _ in range(cfg.n)]
            for rid in resident_ids:
                batches[assignment[rid]].add(rid)
        else:
            batches = sched.initial_partition([requests[rid] for rid in resident_ids], cfg.n)
        state = sched.SchedulerState(n=cfg.n, batches=batches, lengths=lengths, gpu_resident=set(resident_ids),
                                     cpu_pool=set(pool_ids), **knobs)
        ctl = backend.decode_phase(state, cfg, params, requests, metrics, mode, quota)
        next_input = pending[0].input_len if pending else None
        while True:
            if horizon is not None and metrics.iterations >= horizon:
                break
            if next_input is not None and ctl.live_tokens <= cap_tokens and \
                    (ctl.live_tokens + next_input) * cfg.kv_bytes_per_token <= cfg.cpu_kv_capacity:
                break   # resume prefill (REF stop_condition)
            if backend.step(ctl) is None:
                break
        sec = backend.end_decode_phase(ctl)
        metrics.decode_seconds += sec
        clock += sec
        live_tokens = ctl.live_tokens
        ready = sorted(state.lengths)
        if horizon is not None and metrics.iterations >= horizon:
            break

    own_trace.finalize()
    metrics.wall_seconds = clock
    metrics.finalize()
    for r in workload:
        r.generated = requests[r.id].generated
    return metrics
