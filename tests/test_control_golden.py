"""Bit-exact parity of the B200 control plane against golden plan streams
produced by the REFERENCE engine (tests/golden/make_golden.py, which runs
``pipemax.pipeline_sim.simulate_decode`` from the reference checkout).

Every StepPlan field, the scheduler state left by each iteration (batch
membership digests, resident block count, pool size), the reference's block
counts (``GpuState.free_blocks``) and the final metrics must match exactly.
"""
import json
import os

import pytest

from scenarios import scenarios, set_digest

from paper_2605_02189_b200 import scheduler as sched
from paper_2605_02189_b200.control import DecodeControl
from paper_2605_02189_b200.model_core import (ClusterConfig, EstimatorParams, Request,
                                              blocks_for_tokens)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SCEN = scenarios()


def build(sc):
    reqs = {rid: Request(rid, a, b, g) for rid, a, b, g in sc["requests"]}
    cfg = ClusterConfig(**sc["cfg"])
    params = EstimatorParams(*sc["params"])
    resident = list(sc["resident"])
    batches = sched.initial_partition([reqs[r] for r in resident], sc["n"])
    lengths = {rid: r.prefix_len for rid, r in reqs.items()}
    state = sched.SchedulerState(n=sc["n"], batches=batches, lengths=lengths,
                                 gpu_resident=set(resident), cpu_pool=set(reqs) - set(resident),
                                 **sc["knobs"])
    return reqs, cfg, params, state


@pytest.mark.parametrize("name", sorted(SCEN))
def test_plan_stream_matches_reference(name):
    sc = SCEN[name]
    with open(os.path.join(GOLDEN, f"plans_{name}.json")) as fh:
        gold = json.load(fh)
    reqs, cfg, params, state = build(sc)
    ctl = DecodeControl(state, cfg, params, reqs, mode=sc["mode"], quota_tokens=sc["quota"])
    got = []
    for _ in range(sc["horizon"]):
        snap = dict(resident_blocks=state._resident_blocks, pool=len(state.cpu_pool),
                    live=len(state.lengths), batches=[set_digest(b) for b in state.batches],
                    gpu_free=ctl.gpu.free_blocks)
        work = ctl.step()
        if work is None:
            break
        p = work.plan
        rec = {
            "t": p.t, "ijk": [p.exec_batch_index, p.next_batch_index, p.evict_batch_index],
            "exec": set_digest(p.exec_batch), "exec_n": len(p.exec_batch),
            "prefetch": sorted(p.prefetch_set), "evictions": list(p.evictions),
            "residual": set_digest(p.residual), "next": set_digest(p.updated_next_batch),
            "budget": p.prefetch_budget_tokens, "predicted": repr(p.predicted_exec_seconds),
            "steady": p.steady, "residual_tokens": p.residual_tokens,
            "prefetch_tokens": p.prefetch_tokens, **snap,
        }
        got.append(rec)
        # physical pool == reference counts at every iteration boundary
        assert ctl.alloc.free_count == ctl.gpu.free_blocks + ctl.spare_blocks
        for rid, table in ctl.alloc.tables.items():
            assert len(table) == blocks_for_tokens(state.lengths[rid], cfg.block_size)
    assert len(got) == len(gold["records"])
    for a, b in zip(got, gold["records"]):
        assert a == b, f"iteration {b['t']} diverged"
    m, f = ctl.metrics, gold["final"]
    assert m.iterations == f["iterations"]
    assert m.total_tokens_generated == f["total_tokens_generated"]
    assert m.completed_requests == f["completed_requests"]
    assert m.growth_relief_evictions == f["growth_relief_evictions"]
    assert m.steady_iteration == f["steady_iteration"]
    assert [repr(x) for x in m.prefetched_token_fraction] == f["prefetched_token_fraction"]
    assert m.max_resident_tokens == f["max_resident_tokens"]
    assert m.max_active_batch_tokens == f["max_active_batch_tokens"]
    assert repr(m.max_kv_capacity_fraction) == f["max_kv_capacity_fraction"]
    assert ctl.gpu.free_blocks == f["gpu_free_end"]
    assert state._resident_blocks == f["resident_blocks_end"]
    assert {str(r): reqs[r].generated for r in sorted(reqs)} == f["generated"]
