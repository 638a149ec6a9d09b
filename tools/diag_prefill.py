import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from test_engine_gpu import build, oracle_model
spec, eng, reqs, prompts = build()
tt = eng.stages[0][0].tok_table.cpu().numpy()
ref = oracle_model(eng)
for r in range(4):
    caches = ref.new_cache()
    for p, tok in enumerate(prompts[r]):
        lg = ref.token_step(int(tok), p, caches)
    print(r, "engine", tt[eng.slot_of[r]], "oracle", int(np.argmax(lg)), "top3", np.argsort(lg)[-3:], np.sort(lg)[-3:])
