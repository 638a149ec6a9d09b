"""Cluster split-K GEMM (pm_gemm_cl) vs the stream-K kernel + fixup, per
projection shape: R launches over R distinct weights (total > L2) captured in
one CUDA graph and replayed.  Prints us/launch and GB/s of weight bytes, and
(with --sweep) every (slices, clusters) plan of the cluster kernel.

  python tools/gemm_cl_bench.py [M] [model] [--sweep] [--only qkv,o]
"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_02189_b200 import _C, ops  # noqa: E402
from paper_2605_02189_b200.models import SPECS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("M", type=int, nargs="?", default=128)
ap.add_argument("model", nargs="?", default="qwen3-8b")
ap.add_argument("--sweep", action="store_true")
ap.add_argument("--only", default=None)
ap.add_argument("--old", action="store_true", help="also time the stream-K kernel + fixup")
args = ap.parse_args()
dev = "cuda"
s = SPECS[args.model]
M = args.M
shapes = {"qkv": (s.qkv_out, s.d), "o": (s.d, s.H * s.hd), "gate_up": (2 * s.ffn, s.d), "down": (s.d, s.ffn),
          "lm_head": (s.vocab, s.d)}
_C.call("pm_prepare_gemm")
_C.call("pm_prepare_gemm_cl")
st = torch.cuda.Stream()


def timeit(fn, R):
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fn()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            g.replay()
            b.record(st)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3 / R)
    del g
    return best


for name, (n, k) in shapes.items():
    if args.only and name not in args.only.split(","):
        continue
    R = max(4, min(24, int(2.5e9 // (n * k * 2))))
    lins = [ops.Linear((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)) for _ in range(R)]
    m_cap = 128
    x = torch.randn(m_cap, k, device=dev).to(torch.bfloat16)
    maps = ops.activation_maps(x)
    out = torch.zeros(m_cap, n, device=dev, dtype=torch.bfloat16)
    resid = torch.zeros(m_cap, n, device=dev)
    ws = ops.GemmWorkspace(m_cap, ops.GemmWorkspace.floats_needed(lins[:1], m_cap), lins[0].n_units,
                           lins[0].n_units, dev)
    wb = n * k * 2

    def cl_seq(plan=None):
        for lin in lins:
            if plan is not None:
                lin._cl = plan
            if name == "lm_head":
                lin.cl(maps, M, ops.CL_EPI_LOGITS, st, m_cap=m_cap, ws=ws)
            elif name in ("o", "down"):
                lin.cl(maps, M, ops.CL_EPI_RESID, st, m_cap=m_cap, resid=resid)
            elif name == "gate_up":
                lin.cl(maps, M, ops.CL_EPI_SILU, st, m_cap=m_cap, out=out, ld_out=n // 2)
            else:
                lin.cl(maps, M, ops.CL_EPI_STORE, st, m_cap=m_cap, out=out, ld_out=n)

    plan = ops.cl_plan(lins[0].n_units, lins[0].kb)
    t = timeit(cl_seq, R)
    line = (f"{name:8s} [{n}x{k}] M={M}: cluster {t*1e6:7.1f} us {wb/t/1e9:6.0f} GB/s plan(S,NC)={plan} "
            f"ideal@6.55TB/s {wb/6.55e12*1e6:6.1f} us")
    if args.old:
        epi = {"lm_head": ops.EPI_LOGITS_ARGMAX, "o": ops.EPI_RESID_ADD, "down": ops.EPI_RESID_ADD,
               "gate_up": ops.EPI_SILU_MUL, "qkv": ops.EPI_STORE_BF16}[name]

        def old_seq():
            for lin in lins:
                o = resid if epi == ops.EPI_RESID_ADD else (None if epi == ops.EPI_LOGITS_ARGMAX else out)
                lin(maps, M, epi, o, n if epi == ops.EPI_RESID_ADD else (n // 2 if epi == ops.EPI_SILU_MUL else n),
                    ws, st)
        t2 = timeit(old_seq, R)
        line += f" | stream-K+fixup {t2*1e6:7.1f} us {wb/t2/1e9:6.0f} GB/s"
    print(line, flush=True)
    if args.sweep:
        for S in (1, 2, 3, 4):
            cs = 2 * S
            nmax = min(lins[0].n_units, ops.cl_max_clusters(cs))
            cands = sorted({c for c in (nmax, nmax - 1, nmax // 2, lins[0].n_units // 2, lins[0].n_units // 3,
                                        lins[0].n_units // 4, 16, 20, 24, 32) if 1 <= c <= nmax})
            for nc in cands:
                t = timeit(lambda: cl_seq((S, nc)), R)
                print(f"    S={S} NC={nc:3d} ctas={nc*cs:3d} units/cl={-(-lins[0].n_units // nc):3d}: "
                      f"{t*1e6:7.1f} us {wb/t/1e9:6.0f} GB/s", flush=True)
    for lin in lins:
        lin._cl = None
    del lins
    torch.cuda.empty_cache()
