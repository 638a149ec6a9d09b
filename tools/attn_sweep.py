"""Paged attention alone over launch configurations (balanced work split)
on the bench's decode shapes (C2, C3/C4 per-stage rows, C5 points).  CUDA
events around 8 back-to-back launches over different layers (pool >> L2),
median of 5 repeats.  usage: python tools/attn_sweep.py [out.txt]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_02189_b200 import _C, ops  # noqa: E402
from paper_2605_02189_b200.models import LLAMA3_70B, QWEN3_8B, QWEN3_32B  # noqa: E402

dev = "cuda"
_C.call("pm_prepare_attention")
out_f = open(sys.argv[1], "w") if len(sys.argv) > 1 else None


def log(s):
    print(s, flush=True)
    if out_f:
        out_f.write(s + "\n")


g = torch.Generator(device="cpu").manual_seed(0)
shapes = [("C2 qwen3-8b", QWEN3_8B, 36, 128, 768), ("C3 stage qwen3-32b", QWEN3_32B, 8, 48, 1060),
          ("C3 stage qwen3-32b", QWEN3_32B, 8, 64, 1060), ("C4 stage llama3-70b", LLAMA3_70B, 10, 24, 1060),
          ("C4 stage llama3-70b", LLAMA3_70B, 10, 32, 1060), ("C5 qwen3-32b bs256 m4", QWEN3_32B, 16, 64, 1060),
          ("C5 qwen3-32b bs1024 m4", QWEN3_32B, 16, 256, 1060)]
for name, spec, L_s, M, seq in shapes:
    H, Hkv, hd = spec.H, spec.Hkv, spec.hd
    seqs = torch.randint(seq - 64, seq + 64, (M,), generator=g).to(torch.int32)
    nb = (int(seqs.max()) + 15) // 16
    max_blocks = nb + 2
    n_blocks = M * nb + 8
    tok_elems = L_s * 2 * Hkv * hd
    pool = torch.empty(n_blocks * 16 * tok_elems, device=dev, dtype=torch.bfloat16).normal_(0, 0.5)
    perm = torch.randperm(n_blocks)[: M * nb].view(M, nb).to(torch.int32)
    bt = torch.zeros(M, max_blocks, dtype=torch.int32)
    bt[:, :nb] = perm
    bt, seqs_d = bt.to(dev), seqs.to(dev)
    q = torch.randn(M, H, hd, device=dev).to(torch.bfloat16)
    out = torch.empty(M, H, hd, device=dev, dtype=torch.bfloat16)
    tm = ops.pool_tmap(pool, L_s, Hkv, hd)
    kvb = int(seqs.sum()) * 2 * Hkv * hd * 2
    ref = None
    res = []
    for cfg in (1, 2, 0):
        aws = ops.AttnWorkspace(M, Hkv, hd, max_blocks, dev, cfg=cfg)
        aws.set_work(seqs.numpy())
        ts = []
        for rep in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for layer in range(8):
                ops.paged_attention(tm, q, bt, seqs_d, out, aws, M, H, Hkv, hd, layer % L_s, L_s)
            b.record()
            torch.cuda.synchronize()
            if rep:
                ts.append(a.elapsed_time(b) * 1e-3 / 8)
        t = float(np.median(ts))
        if ref is None:
            ref = out.clone()
        err = float((out.float() - ref.float()).abs().max())
        res.append((t, cfg, 0, err))
        log(f"{name:24s} M={M:3d} L_s={L_s:2d} cfg={cfg}: {t*1e6:7.1f} us "
            f"{kvb/t/1e9:6.0f} GB/s  (max|d| vs first {err:.1e})")
    t, cfg, _, _ = min(res)
    log(f"BEST {name} M={M}: cfg={cfg} {t*1e6:.1f} us {kvb/t/1e9:.0f} GB/s")
    del pool
    torch.cuda.empty_cache()
