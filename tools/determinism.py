import sys, os, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_engine_gpu import build
res = []
for rep in range(4):
    spec, eng, reqs, prompts = build(graphs=True)
    for _ in range(40):
        if eng.step() is None: break
    torch.cuda.synchronize()
    res.append(eng.stages[0][0].tok_table[:eng.trash_slot].cpu().tolist())
    del eng
print(os.environ.get("PM_LANES"), os.environ.get("PM_ATTN_CFG"), "slot7:", [r[7] for r in res], "all equal:", all(r == res[0] for r in res))
