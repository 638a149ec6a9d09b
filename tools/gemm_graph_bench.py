"""Steady-state decode GEMM timing: R launches over R distinct weights (total
> L2, so every launch streams from HBM) captured in one CUDA graph and
replayed, like the stage's per-layer sequence.  Prints us/launch and GB/s
of weight bytes per projection shape of Qwen3-8B."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_02189_b200 import _C, ops  # noqa: E402

dev = "cuda"
M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
shapes = {"qkv": (6144, 4096, ops.EPI_STORE_BF16), "o": (4096, 4096, ops.EPI_RESID_ADD),
          "gate_up": (24576, 4096, ops.EPI_SILU_MUL), "down": (4096, 12288, ops.EPI_RESID_ADD),
          "lm_head": (151936, 4096, ops.EPI_LOGITS_ARGMAX)}
_C.call("pm_prepare_gemm")
st = torch.cuda.Stream()
for name, (n, k, epi) in shapes.items():
    if only and name not in only:
        continue
    R = max(4, min(24, int(2.5e9 // (n * k * 2))))
    lins = [ops.Linear((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)) for _ in range(R)]
    x = torch.randn(256, k, device=dev).to(torch.bfloat16)
    maps = ops.activation_maps(x)
    out = torch.zeros(256, n, device=dev, dtype=torch.float32)
    ws = ops.GemmWorkspace(256, ops.GemmWorkspace.floats_needed(lins[:1], 256), lins[0].n_units, lins[0].n_units, dev)
    o = out if epi != ops.EPI_LOGITS_ARGMAX else None
    pf_mb = float(os.environ.get("PF_MB", "0"))

    def seq():
        for i, lin in enumerate(lins):
            nxt = lins[(i + 1) % len(lins)]
            pf = (nxt.packed, min(nxt.packed.numel() * 2, int(pf_mb * 2**20))) if pf_mb > 0 else None
            lin(maps, M, epi, o, n, ws, st, prefetch=pf)
    with torch.cuda.stream(st):
        seq()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        seq()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            g.replay()
            b.record(st)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3 / R)
    print(f"{name:8s} [{n}x{k}] M={M} R={R}: {best*1e6:7.1f} us/launch  {n*k*2/best/1e9:6.0f} GB/s  "
          f"ideal@6.65TB/s {n*k*2/6.65e12*1e6:6.1f} us  plan={lins[0].plan(M)}")
    del lins, g
    torch.cuda.empty_cache()
