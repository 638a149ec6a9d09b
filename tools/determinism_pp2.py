"""Run-to-run determinism of the single-process PP=2 engine (graphs) on the
two-rank test's scenario: per-step greedy ids of the last stage, 5 repeats;
reports zero / diverging ids."""
import os, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_pipeline_gpu import _scenario
from paper_2605_02189_b200.engine import DecodeEngine
logs = []
for rep in range(int(os.environ.get("REPS", "5"))):
    spec, st, cfg, params, reqs = _scenario()
    ref = DecodeEngine(spec, st, cfg, params, reqs, pp=2, kv_init="random", seed=5, graphs=True)
    log = []
    for n in range(60):
        w = ref.step()
        if w is None: break
        if w.rows:
            torch.cuda.synchronize()
            log.append((n, list(w.rows), ref.stages[-1][0].out_ids[:len(w.rows)].cpu().tolist()))
    logs.append(log)
    del ref
    torch.cuda.synchronize()
bad = [next(((a, b) for a, b in zip(l, logs[0]) if a != b), None) for l in logs]
zeros = [sum(1 for _, _, ids in l for x in ids if x == 0) for l in logs]
print(os.environ.get("PM_PDL"), "zero ids per run:", zeros, "first divergence vs run 0:", [b[0][:1] if b else None for b in bad])
