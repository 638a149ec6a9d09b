"""Per-CTA globaltimer trace of one decode GEMM launch (PM_GEMM_DEBUG=8):
start, end of segment loop, and for up to two split units: counter wait
done, partial slices staged, fixup done (ns, relative to the first CTA)."""
import ctypes as C
import os
import sys

os.environ["PM_GEMM_DEBUG"] = "8"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2605_02189_b200 import _C, ops  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
M = int(sys.argv[3]) if len(sys.argv) > 3 else 128
epi = int(sys.argv[4]) if len(sys.argv) > 4 else ops.EPI_STORE_BF16
dev = "cuda"
_C.call("pm_prepare_gemm")
lins = [ops.Linear((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)) for _ in range(8)]
x = torch.randn(256, k, device=dev).to(torch.bfloat16)
maps = ops.activation_maps(x)
out = torch.zeros(256, n, device=dev, dtype=torch.float32)
ws = ops.GemmWorkspace(256, ops.GemmWorkspace.floats_needed(lins[:1], 256), lins[0].n_units, lins[0].n_units, dev)
for _ in range(3):
    for lin in lins:
        lin(maps, M, epi, out, n, ws)
torch.cuda.synchronize()
buf = np.zeros(148 * 8, dtype=np.uint64)
_C.lib().pm_gemm_trace_read.argtypes = [C.c_void_p]
_C.lib().pm_gemm_trace_read(buf.ctypes.data_as(C.c_void_p))
t = buf.reshape(148, 8).astype(np.int64)
t0 = t[:, 0].min()
rel = np.where(t > 0, t - t0, -1)
print(f"shape {n}x{k} M={M} plan={lins[0].plan(M)}")
print("cta   start  waited lastmma  epi_end (us)")
for c in list(range(0, 148, 9)) + [147]:
    print(f"{c:3d} " + " ".join(f"{v/1e3:7.1f}" if v >= 0 else "      -" for v in rel[c, :4]))
for k, name in [(1, "waited"), (2, "last mma"), (3, "epilogue end")]:
    v = rel[:, k][rel[:, k] >= 0]
    print(f"{name:13s} min {v.min()/1e3:7.1f} median {np.median(v)/1e3:7.1f} max {v.max()/1e3:7.1f}")

sm = t[:, 4]
lm = rel[:, 2]
order = np.argsort(sm)
print("last-mma (us) by SM id (sorted):")
for k in range(0, 148, 8):
    idx = order[k:k + 8]
    print(" ".join(f"{int(sm[i]):3d}:{lm[i] / 1e3:5.1f}" for i in idx))
