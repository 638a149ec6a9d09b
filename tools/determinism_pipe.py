"""Run-to-run determinism of the PipelineRank step path (world size 1) on the
tiny engine scenario: slot 7's token after 40 steps, 4 repeats."""
import os, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_engine_gpu import build
from paper_2605_02189_b200.pipeline import PipelineRank
res = []
for rep in range(4):
    spec, eng2, reqs2, prompts2 = build(graphs=True)
    ex, kv = eng2.stages[0]
    class _Fwd:
        resid, out_ids, tok_table = ex.resid, ex.out_ids, ex.tok_table
        def forward(self_, M):
            ex.run(M, kv.compute, graphs=eng2.graphs)
    pr = PipelineRank(eng2.control, _Fwd(), eng2.slot_of, rank=0, world=1, kv=kv,
                      upload_meta=lambda rows, pos, tab: eng2._upload_meta(rows, pos, tab, stream=kv.compute),
                      stream=kv.compute, bucket=eng2.bucket)
    for _ in range(40):
        if pr.step() is None: break
    pr.finish(); torch.cuda.synchronize()
    res.append(ex.tok_table[:eng2.trash_slot].cpu().tolist())
    del eng2, pr
print(os.environ.get("PM_PDL"), os.environ.get("PM_OFFLOAD_MODE"), "slot7:", [r[7] for r in res],
      "diff slots vs first:", [[i for i in range(len(r)) if r[i] != res[0][i]] for r in res])
