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
