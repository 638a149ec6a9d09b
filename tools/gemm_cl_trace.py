"""Per-CTA timeline of one cluster-GEMM launch (PM_CL_TRACE=1 globaltimer
stamps): prints, relative to the earliest CTA start, the median / max over
CTAs of each stamp (setup, first weights, last MMA, first partial, partials
ready, epilogue done, exit).

  PM_CL_TRACE=1 python tools/gemm_cl_trace.py [n_out k M S NC]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("PM_CL_TRACE", "1")
from paper_2605_02189_b200 import _C, ops  # noqa: E402

n, k, M = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (6144, 4096, 128)
plan = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else None
dev = "cuda"
lins = [ops.Linear((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)) for _ in range(4)]
x = torch.randn(128, k, device=dev).to(torch.bfloat16)
maps = ops.activation_maps(x)
out = torch.zeros(128, n, device=dev, dtype=torch.bfloat16)
for rep in range(3):
    for lin in lins:
        if plan:
            lin._cl = plan
        lin.cl(maps, M, ops.CL_EPI_STORE, m_cap=128, out=out, ld_out=n)
torch.cuda.synchronize()
buf = np.zeros(160 * 8, dtype=np.uint64)
_C.call("pm_gemm_cl_trace_read", _C.C.c_void_p(buf.ctypes.data))
S, nc = lins[-1]._cl
ctas = nc * 2 * S
t = buf.reshape(160, 8)[:ctas].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["start", "setup", "first_w", "last_mma", "first_part", "parts_ready", "epi_done", "exit"]
print(f"[{n}x{k}] M={M} plan S={S} NC={nc} ctas={ctas} weight bytes/CTA={n * k * 2 / ctas / 1e6:.2f} MB")
for i, nm in enumerate(names):
    col = rel[:, i]
    print(f"  {nm:12s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
