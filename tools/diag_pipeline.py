"""Diagnostic: per-step greedy ids of the single-process PP=2 engine on the
two-rank test scenario (tests/test_pipeline_gpu.py), printed for the first
steps; run it twice in fresh processes to check run-to-run determinism."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_pipeline_gpu import _scenario  # noqa: E402

from paper_2605_02189_b200.engine import DecodeEngine  # noqa: E402

spec, st, cfg, params, reqs = _scenario()
pp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ref = DecodeEngine(spec, st, cfg, params, reqs, pp=pp, kv_init="random", seed=5, graphs=True)
print("numa", ref.stages[0][1].rep.numa_node, "pool sums", [float(ex.pool.float().abs().sum()) for ex, _ in ref.stages])
for n in range(4):
    w = ref.step()
    torch.cuda.synchronize()
    print(n, w.rows, w.positions, ref.stages[-1][0].out_ids[:len(w.rows)].cpu().tolist(),
          "prefetch", [p[0] for p in w.prefetch])
