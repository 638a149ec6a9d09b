"""The reference's own decode loop on B200 transfers (paper_2605_02189_b200/seam.py).

The UNMODIFIED reference engine ``pipemax.pipeline_sim._DecodeEngine`` (REF
pipeline_sim.py:330-543, installed from /root/reference into baseline/_ref --
skipped when that install is absent) runs with ``B200GpuState`` as its
``gpu`` and ``B200CopyChannel`` as its ``h2d``/``d2h`` links:
  * its plan stream and outcome equal the reference's own ``simulate_decode``
    (iterations, completions, tokens; the loop's decisions never read time);
  * the block counts it sees every step equal the reference ``GpuState``'s
    (the physical allocator mirrors them);
  * every ``kv_prefetch`` stream really lands the request's host-replica
    blocks in the physical blocks the allocator gave it (byte-exact), and the
    bytes moved equal the reference's per-block chunk arithmetic;
  * the loop's stall/transfer accounting now rests on measured copy times."""
import copy
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def pm():
    if not os.path.isdir(os.path.join(REF, "pipemax")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import pipemax
        from pipemax import model_core, pipeline_sim
        for name in ("blocks_for_tokens", "capacity_blocks"):
            if not hasattr(pipemax, name):
                setattr(pipemax, name, getattr(model_core, name))
        yield pipemax, pipeline_sim
    finally:
        sys.path.remove(REF)


def _scenario(pm, n_req=40, m=4, seed=1):
    rng = np.random.default_rng(seed)
    reqs = {i: pm.Request(i, int(rng.integers(20, 90)), int(rng.integers(8, 30))) for i in range(n_req)}
    resident = list(range(16))
    batches = pm.initial_partition([reqs[r] for r in resident], m)
    st = pm.SchedulerState(n=m, batches=batches, lengths={r: q.prefix_len for r, q in reqs.items()},
                           gpu_resident=set(resident), cpu_pool=set(reqs) - set(resident), ema_alpha=0.3,
                           window_w=3, stability_threshold=0.5)
    kv = 8192
    cap_blocks = sum(pm.blocks_for_tokens(reqs[r].input_len, 16) for r in resident) + 12
    cfg = pm.ClusterConfig(n=m, mem_per_gpu=-(-cap_blocks * 16 * kv // m), model_bytes=0, kv_bytes_per_token=kv,
                           h2d_bandwidth=5e9, d2h_bandwidth=5e9, cpu_kv_capacity=10**15, block_size=16)
    params = pm.EstimatorParams(1e-5, 1e-8, 2e-4)
    return reqs, st, cfg, params


def test_reference_loop_drives_b200_copies(pm):
    pmx, ps = pm
    from paper_2605_02189_b200.kv import HostReplica
    from paper_2605_02189_b200.seam import B200CopyChannel, B200GpuState

    reqs, st, cfg, params = _scenario(pmx)
    # the reference's own run (simulated links) on a copy of the same state
    want_trace, want = ps.simulate_decode(copy.deepcopy(st), cfg, params, None, None,
                                          requests=copy.deepcopy(reqs), seed=0)

    st.configure_blocks(cfg.block_size)
    cap = pmx.capacity_blocks(cfg)
    block_bytes = int(cfg.block_size * cfg.kv_bytes_per_token / cfg.n)   # the reference's chunk_bytes
    gpu = B200GpuState(0, cap, cap - st.resident_blocks())
    for rid in sorted(st.gpu_resident):
        gpu.seed(rid, pmx.blocks_for_tokens(st.lengths[rid], cfg.block_size))
    slot_of = {r: i for i, r in enumerate(sorted(reqs))}
    max_blocks = max(pmx.blocks_for_tokens(q.input_len + q.output_len + 1, 16) for q in reqs.values())
    rep = HostReplica(len(reqs), max_blocks, block_bytes, numa_node=-1)
    host = rep.as_tensor()
    host.copy_(torch.randint(0, 256, (host.numel(),), dtype=torch.uint8, generator=torch.Generator().manual_seed(2)))
    dev = torch.device("cuda")
    pool = torch.zeros(cap * block_bytes, dtype=torch.uint8, device=dev)
    for rid in st.gpu_resident:
        for lb, pb in enumerate(gpu.blocks_of(rid)):
            o = rep.offset(slot_of[rid], lb)
            pool[pb * block_bytes:(pb + 1) * block_bytes].copy_(host[o:o + block_bytes])
    h2d = B200CopyChannel("h2d", pool=pool, replica=rep, slot_of=slot_of, gpu=gpu, block_bytes=block_bytes,
                          name="h2d0")
    d2h = B200CopyChannel("d2h", pool=pool, replica=rep, slot_of=slot_of, gpu=gpu, block_bytes=block_bytes,
                          name="d2h0")
    trace, metrics = ps.EventTrace(), ps.EpisodeMetrics()
    counts, landed = [], []
    real_grow, real_copy = gpu.grow, h2d._prefetch_copy

    def grow(rid):   # watch the counts the loop sees at every block crossing
        real_grow(rid)
        counts.append(dict(gpu.resident_blocks) == {r: len(b) for r, b in gpu.alloc.tables.items()})

    def prefetch_copy(rid):   # every prefetch lands the request's replica blocks, byte for byte
        n = real_copy(rid)
        torch.cuda.current_stream().synchronize()
        ok = True
        for lb, pb in enumerate(gpu.blocks_of(rid)):
            o = rep.offset(slot_of[rid], lb)
            ok &= torch.equal(pool[pb * block_bytes:(pb + 1) * block_bytes].cpu(), host[o:o + block_bytes])
        landed.append(ok)
        return n
    gpu.grow, h2d._prefetch_copy = grow, prefetch_copy
    eng = ps._DecodeEngine(st, cfg, params, None, np.random.default_rng([0, 1]), reqs, trace, metrics, gpu, h2d, d2h)
    eng.run()
    h2d.drain()
    d2h.drain()
    torch.cuda.synchronize()

    assert metrics.iterations == want.iterations
    assert metrics.completed_requests == want.completed_requests == len(reqs)
    assert metrics.total_tokens_generated == want.total_tokens_generated
    assert counts and all(counts), "physical tables diverged from the block counts"
    pre = [r for r in h2d.records if isinstance(r.tag, tuple) and r.tag[0] == "kv_prefetch"]
    assert pre and landed and all(landed)
    # bytes moved = blocks x chunk_bytes, the reference's per-request stream arithmetic
    assert all(r.n_bytes == r.chunks * block_bytes for r in pre)
    assert all(r.end >= r.start >= r.queued_at - 1e-12 for r in h2d.records + d2h.records)
    assert metrics.stall_seconds >= 0.0
