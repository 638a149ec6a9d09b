"""Generate golden plan/residency streams by running the REFERENCE decode
engine (``pipemax.pipeline_sim.simulate_decode``) on every scenario of
``scenarios.py``.

Run in the build container, where the reference is mounted read-only:

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

It wraps the reference's ``scheduler._plan_step`` (the engine calls it through
the module attribute, REF pipeline_sim.py:402) to capture every StepPlan and a
snapshot of the scheduler state at plan time, and subclasses ``GpuState``
(REF pipeline_sim.py:121-153) to capture block counts.  Output:
``tests/golden/plans_<scenario>.json`` -- committed; the GPU box never needs
the reference.
"""

import argparse
import importlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from scenarios import scenarios, set_digest  # noqa: E402


def plan_record(plan, state, gpu):
    return {
        "t": plan.t,
        "ijk": [plan.exec_batch_index, plan.next_batch_index, plan.evict_batch_index],
        "exec": set_digest(plan.exec_batch),
        "exec_n": len(plan.exec_batch),
        "prefetch": sorted(plan.prefetch_set),
        "evictions": list(plan.evictions),
        "residual": set_digest(plan.residual),
        "next": set_digest(plan.updated_next_batch),
        "budget": plan.prefetch_budget_tokens,
        "predicted": repr(plan.predicted_exec_seconds),
        "steady": plan.steady,
        "residual_tokens": plan.residual_tokens,
        "prefetch_tokens": plan.prefetch_tokens,
        # state as the previous iteration left it
        "resident_blocks": state._resident_blocks,
        "pool": len(state.cpu_pool),
        "live": len(state.lengths),
        "batches": [set_digest(b) for b in state.batches],
        "gpu_free": gpu.free_blocks if gpu is not None else None,
    }


def run(ref_src):
    sys.path.insert(0, ref_src)
    pm = importlib.import_module("pipemax")
    ps = importlib.import_module("pipemax.pipeline_sim")
    sch = importlib.import_module("pipemax.scheduler")
    mc = importlib.import_module("pipemax.model_core")
    assert os.path.realpath(pm.__file__).startswith(os.path.realpath(ref_src)), pm.__file__

    for name, sc in scenarios().items():
        gpus = []

        base_gpu = ps.GpuState

        class TracedGpu(base_gpu):
            def __init__(self, *a, **kw):
                super().__init__(*a, **kw)
                gpus.append(self)

        records = []
        orig = sch._plan_step

        def traced(state, params, cfg, mode="dynamic", quota_tokens=0):
            plan = orig(state, params, cfg, mode=mode, quota_tokens=quota_tokens)
            records.append(plan_record(plan, state, gpus[-1] if gpus else None))
            return plan

        reqs = {rid: mc.Request(rid, a, b, g) for rid, a, b, g in sc["requests"]}
        cfg = mc.ClusterConfig(**sc["cfg"])
        params = mc.EstimatorParams(*sc["params"])
        resident = list(sc["resident"])
        batches = sch.initial_partition([reqs[r] for r in resident], sc["n"])
        lengths = {rid: r.prefix_len for rid, r in reqs.items()}
        pool = set(reqs) - set(resident)
        state = sch.SchedulerState(n=sc["n"], batches=batches, lengths=lengths,
                                   gpu_resident=set(resident), cpu_pool=pool, **sc["knobs"])
        sch._plan_step = traced
        ps.GpuState = TracedGpu
        try:
            if sc["mode"] == "dynamic":
                _, metrics = ps.simulate_decode(state, cfg, params, ps.NoiseSpec("none"),
                                                sc["horizon"], requests=reqs, seed=0)
            else:
                # simulate_decode is dynamic-only; drive the engine class
                # directly for the baseline policies (REF :330-356).
                import numpy as np
                trace, metrics = ps.EventTrace(), ps.EpisodeMetrics()
                state.configure_blocks(cfg.block_size)
                cap = mc.capacity_blocks(cfg)
                gpu = TracedGpu(0, cap, cap - state.resident_blocks())
                for rid in state.gpu_resident:
                    gpu.resident_blocks[rid] = mc.blocks_for_tokens(state.lengths[rid], cfg.block_size)
                h2d = ps.ChannelSim("h2d", cfg.h2d_bandwidth, 0.0, True, name="h2d0")
                d2h = ps.ChannelSim("d2h", cfg.d2h_bandwidth, 0.0, True, name="d2h0")
                eng = ps._DecodeEngine(state, cfg, params, ps.NoiseSpec("none"),
                                       np.random.default_rng([0, 1]), reqs, trace, metrics,
                                       gpu, h2d, d2h, mode=sc["mode"], quota_tokens=sc["quota"])
                eng.run(horizon=sc["horizon"])
        finally:
            sch._plan_step = orig
            ps.GpuState = base_gpu
        final = {
            "iterations": metrics.iterations,
            "total_tokens_generated": metrics.total_tokens_generated,
            "completed_requests": metrics.completed_requests,
            "growth_relief_evictions": metrics.growth_relief_evictions,
            "steady_iteration": metrics.steady_iteration,
            "prefetched_token_fraction": [repr(x) for x in metrics.prefetched_token_fraction],
            "max_resident_tokens": metrics.max_resident_tokens,
            "max_active_batch_tokens": metrics.max_active_batch_tokens,
            "max_kv_capacity_fraction": repr(metrics.max_kv_capacity_fraction),
            "gpu_free_end": gpus[-1].free_blocks,
            "resident_blocks_end": state._resident_blocks,
            "generated": {str(r): reqs[r].generated for r in sorted(reqs)},
        }
        path = os.path.join(HERE, f"plans_{name}.json")
        with open(path, "w") as fh:
            json.dump({"scenario": name, "records": records, "final": final}, fh,
                      separators=(",", ":"))
        n_pf = sum(len(r["prefetch"]) for r in records)
        n_ev = sum(len(r["evictions"]) for r in records)
        print(f"{name}: {len(records)} plans, {n_pf} prefetches, {n_ev} evictions, "
              f"{metrics.growth_relief_evictions} relief, {metrics.completed_requests} done, "
              f"steady@{metrics.steady_iteration} -> {os.path.getsize(path)//1024} KiB")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    run(ap.parse_args().ref)
