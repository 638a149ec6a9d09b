"""Time the decode GEMM on the Qwen3-8B projection shapes (CUDA events, L2
flushed between launches) for a few K-splits; prints GB/s of weight bytes."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_02189_b200 import ops  # noqa: E402

dev = "cuda"
M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
shapes = {"qkv": (6144, 4096, ops.EPI_STORE_BF16), "o": (4096, 4096, ops.EPI_RESID_ADD),
          "gate_up": (24576, 4096, ops.EPI_SILU_MUL), "down": (4096, 12288, ops.EPI_RESID_ADD),
          "lm_head": (151936, 4096, ops.EPI_LOGITS_ARGMAX)}
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name, (n, k, epi) in shapes.items():
    w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    x = torch.randn(256, k, device=dev).to(torch.bfloat16)
    maps = ops.activation_maps(x)
    out = torch.zeros(256, n, device=dev, dtype=torch.float32)
    lin = ops.Linear(w)
    ws = ops.GemmWorkspace(256, ops.GemmWorkspace.floats_needed([lin], 256), lin.n_units, lin.n_units, dev)
    res = []
    for s in [0]:
        times = []
        for it in range(8):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lin(maps, M, epi, out if epi != ops.EPI_LOGITS_ARGMAX else None, n, ws)
            b.record()
            torch.cuda.synchronize()
            if it >= 2:
                times.append(a.elapsed_time(b) * 1e-3)
        t = min(times)
        res.append(f"{t*1e6:7.1f}us {n*k*2/t/1e9:6.0f}GB/s plan={lin.plan(M)}")
    print(f"{name:8s} [{n}x{k}] M={M}: " + " | ".join(res))
