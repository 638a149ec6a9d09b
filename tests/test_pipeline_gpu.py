"""The rank-per-stage pipeline driver (pipeline.PipelineEngine) on one GPU
with world size 1: the PipelineRank step path (replicated control plane, KV
engine, stage CUDA graphs, no P2P) produces exactly the tokens of the
single-process DecodeEngine (two lanes in flight) for the same plan stream.  (The NCCL P2P schedule
itself is covered by the gloo world-size-2 tests.)"""
import pytest
import torch

from paper_2605_02189_b200.pipeline import PipelineRank
from test_engine_gpu import build  # noqa: E402

pytestmark = pytest.mark.gpu


def test_pipeline_world1_matches_engine():
    spec, ref, reqs, prompts = build(graphs=True)
    for _ in range(40):
        if ref.step() is None:
            break
    torch.cuda.synchronize()
    # real request slots only: the trailing trash slot takes whatever the
    # graph bucket's padding rows write (undefined by design)
    want = ref.stages[0][0].tok_table[:ref.trash_slot].clone()
    # same scenario through the pipeline driver (prefill seeds the same KV)
    spec2, eng2, reqs2, prompts2 = build(graphs=True)
    # wrap the prefilled engine exactly as PipelineEngine does for its stage
    ex, kv = eng2.stages[0]

    class _Fwd:
        resid, out_ids, tok_table = ex.resid, ex.out_ids, ex.tok_table

        def forward(self_, M):
            ex.run(M, kv.compute, graphs=eng2.graphs)
    pr = PipelineRank(eng2.control, _Fwd(), eng2.slot_of, rank=0, world=1, kv=kv,
                      upload_meta=lambda rows, pos, tab: eng2._upload_meta(rows, pos, tab, stream=kv.compute),
                      stream=kv.compute, bucket=eng2.bucket)
    for _ in range(40):
        if pr.step() is None:
            break
    pr.finish()
    torch.cuda.synchronize()
    assert torch.equal(ex.tok_table[:eng2.trash_slot], want)


def _two_rank_worker(rank, world, port, q, n_steps):
    import os
    import torch.distributed as dist
    from paper_2605_02189_b200.pipeline import PipelineEngine, make_groups
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, st, cfg, params, reqs = _scenario()
        peng = PipelineEngine(spec, st, cfg, params, reqs, rank=rank, world=world, device="cuda:0",
                              kv_init="random", seed=5, transport="staged", groups=make_groups(world))
        n, ids_log = 0, []
        while n < n_steps:
            w = peng.step()
            if w is None:
                break
            if rank == world - 1 and w.rows:
                torch.cuda.synchronize()
                ids_log.append((n, list(w.rows), peng.ex.out_ids[:len(w.rows)].cpu().tolist()))
            n += 1
        peng.finish()
        torch.cuda.synchronize()
        digests = [None] * world
        dist.all_gather_object(digests, peng.pr.digests)
        assert all(d == digests[0] for d in digests), "replicated plan streams diverged"
        if rank == 0:
            q.put(("ok", peng.ex.tok_table[:len(reqs)].cpu().tolist(), n))
        if rank == world - 1:
            q.put(("ids", ids_log, n))
        dist.barrier()
    except Exception as e:
        q.put(("err", repr(e), 0))
        raise
    finally:
        dist.destroy_process_group()


def _scenario():
    import numpy as np
    from paper_2605_02189_b200 import scheduler as sched
    from paper_2605_02189_b200.models import TINY
    from test_engine_gpu import _cap_cfg
    from paper_2605_02189_b200.model_core import EstimatorParams, Request
    rng = np.random.default_rng(9)
    reqs = {i: Request(i, int(rng.integers(17, 41)), int(rng.integers(6, 16))) for i in range(24)}
    resident = list(range(12))
    m = 4
    batches = sched.initial_partition([reqs[r] for r in resident], m)
    st = sched.SchedulerState(n=m, batches=batches, lengths={r: q.prefix_len for r, q in reqs.items()},
                              gpu_resident=set(resident), cpu_pool=set(reqs) - set(resident),
                              ema_alpha=0.3, window_w=3, stability_threshold=0.5)
    return TINY, st, _cap_cfg(m, 40, TINY.kv_bytes_per_token()), EstimatorParams(1e-6, 2e-8, 1e-4), reqs


def test_pipeline_two_ranks_one_gpu_matches_single_process():
    """The rank-per-stage pipeline with TWO processes on one B200 (stage 0 and
    stage 1 of a PP=2 split, activations bf16 over the staged gloo transport,
    ids last -> first on their own process group, stage-0 scatter from mapped
    slots): the token table equals the single-process PP=2 engine's, which
    applies the same bf16 hop between its two local stages."""
    import socket
    import torch.multiprocessing as mp
    from paper_2605_02189_b200.engine import DecodeEngine
    n_steps = 60
    spec, st, cfg, params, reqs = _scenario()
    ref = DecodeEngine(spec, st, cfg, params, reqs, pp=2, kv_init="random", seed=5, graphs=True)
    n, ref_log = 0, []
    while n < n_steps:
        w = ref.step()
        if w is None:
            break
        if w.rows:
            torch.cuda.synchronize()
            ref_log.append((n, list(w.rows), ref.stages[-1][0].out_ids[:len(w.rows)].cpu().tolist()))
        n += 1
    torch.cuda.synchronize()
    single = ref.stages[0][0].tok_table[:len(reqs)].cpu().tolist()
    # the token table every step's ids imply (first tokens, then each step's greedy ids in step order)
    spec2, st2, cfg2, params2, reqs2 = _scenario()
    ref2 = DecodeEngine(spec2, st2, cfg2, params2, reqs2, pp=2, kv_init="none", seed=5, graphs=False)
    want = ref2.stages[0][0].tok_table[:len(reqs)].cpu().tolist()
    del ref2
    for _, rows, ids in ref_log:
        for r, i in zip(rows, ids):
            want[ref.slot_of[r]] = i
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q, n_steps)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        kind, payload, steps = q.get(timeout=600)
        got[kind] = (payload, steps)
    for p in procs:
        p.join(timeout=120)
    assert "err" not in got, got.get("err")
    table, steps = got["ok"]
    ids_log, _ = got["ids"]
    assert steps == n
    first_bad = next(((a, b) for a, b in zip(ids_log, ref_log) if a != b), None)
    assert first_bad is None, f"first diverging step (pipeline, single-process): {first_bad}"
    assert single == want, [i for i in range(len(want)) if single[i] != want[i]]
    assert table == want, [i for i in range(len(want)) if table[i] != want[i]]
