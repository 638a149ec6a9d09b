"""Golden plan streams of the REFERENCE episode runner
(``pipemax.pipeline_sim.run_episode``, REF pipeline_sim.py:604-780) on the
scenarios of ``episode_scenarios.py``: every StepPlan (through the wrapped
``scheduler._plan_step``), every phase switch and the final metrics.

    python tests/golden/make_episode_golden.py [--ref /root/reference/pkg/src]
"""

import argparse
import importlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from episode_scenarios import episode_scenarios  # noqa: E402
from scenarios import set_digest  # noqa: E402


def plan_record(plan, state):
    return {"t": plan.t, "ijk": [plan.exec_batch_index, plan.next_batch_index, plan.evict_batch_index],
            "exec": set_digest(plan.exec_batch), "prefetch": sorted(plan.prefetch_set),
            "evictions": list(plan.evictions), "budget": plan.prefetch_budget_tokens, "steady": plan.steady,
            "resident": sorted(state.gpu_resident), "pool": len(state.cpu_pool), "live": len(state.lengths)}


def run(ref_src):
    sys.path.insert(0, ref_src)
    ps = importlib.import_module("pipemax.pipeline_sim")
    sch = importlib.import_module("pipemax.scheduler")
    mc = importlib.import_module("pipemax.model_core")
    for name, sc in episode_scenarios().items():
        records = []
        orig = sch._plan_step

        def traced(state, params, cfg, mode="dynamic", quota_tokens=0):
            plan = orig(state, params, cfg, mode=mode, quota_tokens=quota_tokens)
            records.append(plan_record(plan, state))
            return plan
        workload = [mc.Request(rid, a, b, g) for rid, a, b, g in sc["requests"]]
        cfg = mc.ClusterConfig(**sc["cfg"])
        params = mc.EstimatorParams(*sc["params"])
        trace = ps.EventTrace()
        sch._plan_step = traced
        try:
            m = ps.run_episode(workload, cfg, params, policy=sc["policy"], seed=0, noise_spec=ps.NoiseSpec("none"),
                               scheduler_knobs=dict(sc["knobs"]), rho_hi=sc["rho_hi"], horizon=sc["horizon"],
                               trace=trace)
        finally:
            sch._plan_step = orig
        switches = [[ev.payload["to"], ev.payload["live_kv_tokens"]] for ev in trace.events
                    if ev.kind == "phase_switch"]
        final = {"iterations": m.iterations, "total_tokens_generated": m.total_tokens_generated,
                 "completed_requests": m.completed_requests, "phase_switches": m.phase_switches,
                 "growth_relief_evictions": m.growth_relief_evictions,
                 "generated": {str(r.id): r.generated for r in workload}}
        path = os.path.join(HERE, f"episode_{name}.json")
        with open(path, "w") as fh:
            json.dump({"scenario": name, "records": records, "switches": switches, "final": final}, fh,
                      separators=(",", ":"))
        print(f"{name}: {len(records)} plans, {m.phase_switches} phase switches, "
              f"{m.completed_requests} done -> {os.path.getsize(path) // 1024} KiB")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    run(ap.parse_args().ref)
