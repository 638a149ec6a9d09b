"""Prefill with layer-wise async KV offload (prefill.py; REF
pipeline_sim.py:241-323): the host replica a request ends with does not
depend on whether it was prefilled into its own (resident) blocks or through
a bounded staging area; resident requests' HBM blocks equal their host copy;
the trace carries one offload transfer per (request, chunk, layer, stage) and
backpressure stalls when staging is bounded to one request.  Numerical
correctness of the prefill output is covered by test_engine_gpu (first
generated token and every later logit vs the fp32 oracle)."""
import numpy as np
import pytest
import torch

from paper_2605_02189_b200.prefill import run_prefill
from test_engine_gpu import build  # noqa: E402  (tests/ is on sys.path via rootdir conftest)

pytestmark = pytest.mark.gpu


def _replica_prefix(kv, slot, n_tokens, tok_bytes):
    host = kv.rep.as_tensor()
    off = kv.rep.offset(slot)
    return host[off:off + n_tokens * tok_bytes].clone()


@pytest.mark.parametrize("pp", [1, 2])
def test_prefill_replica_independent_of_residency(pp):
    spec, eng_a, reqs, prompts = build(pp=pp, graphs=False)
    torch.cuda.synchronize()
    cfg, params = eng_a.cfg, eng_a.params
    trace, makespan, eng_b = run_prefill(reqs, prompts, cfg, params, spec, pp=pp, staging_pool_requests=1,
                                         seed=3, graphs=False)
    assert makespan > 0
    for si in range(pp):
        ex_a, kv_a = eng_a.stages[si]
        ex_b, kv_b = eng_b.stages[si]
        tb = ex_a.tok_bytes
        pool_a = ex_a.pool.view(torch.uint8).view(ex_a.pool_blocks, ex_a.block_bytes)
        for rid, q in reqs.items():
            L = q.input_len
            ha = _replica_prefix(kv_a, eng_a.slot_of[rid], L, tb)
            hb = _replica_prefix(kv_b, eng_b.slot_of[rid], L, tb)
            assert torch.equal(ha, hb), f"stage {si} request {rid}: host replicas differ"
            table = eng_a.control.alloc.tables.get(rid)
            if table is not None:   # resident in A: its blocks hold the same bytes
                dev = torch.cat([pool_a[b] for b in table]).cpu()[:L * tb]
                assert torch.equal(dev, ha), f"stage {si} request {rid}: HBM != host"
    # first generated token identical either way
    assert torch.equal(eng_a.stages[0][0].tok_table[:len(reqs)].cpu(), eng_b.stages[0][0].tok_table[:len(reqs)].cpu())


def test_prefill_trace_offload_events_and_backpressure():
    spec, eng, reqs, prompts = build(graphs=False)
    trace, makespan, eng_b = run_prefill(reqs, prompts, eng.cfg, eng.params, spec, staging_pool_requests=1,
                                         seed=3, graphs=False)
    m_cap = eng_b.m_cap
    chunks = sum(-(-q.input_len // m_cap) for q in reqs.values())
    starts = trace.select("transfer_start")
    assert len(starts) == chunks * spec.layers
    assert {e.payload["layer"] for e in starts} == set(range(spec.layers))
    assert len(trace.select("stage_compute_start")) == chunks
    # one staging area: every pooled request after the first waits on the previous one's offload
    assert len(trace.select("stall_start")) == len(reqs) - 1
    ends = trace.select("transfer_end")
    assert max(e.time for e in ends) <= makespan + 1e-9
