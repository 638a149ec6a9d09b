"""Per-warp globaltimer trace of one paged-attention launch (PM_ATTN_DEBUG=4):
distribution of warp start, first-data and end times and blocks per warp."""
import ctypes as C
import os
import sys

os.environ["PM_ATTN_DEBUG"] = str(4 | int(os.environ.get("EXTRA_DEBUG", "0")))
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2605_02189_b200 import _C, ops  # noqa: E402
from paper_2605_02189_b200.models import SPECS  # noqa: E402

dev = "cuda"
# usage: attn_trace.py [seq] [model] [L_s] [M]
seq = int(sys.argv[1]) if len(sys.argv) > 1 else 550
spec = SPECS[sys.argv[2]] if len(sys.argv) > 2 else SPECS["qwen3-8b"]
L_s = int(sys.argv[3]) if len(sys.argv) > 3 else 36
M = int(sys.argv[4]) if len(sys.argv) > 4 else 128
H, Hkv, hd = spec.H, spec.Hkv, spec.hd
g = torch.Generator(device=dev).manual_seed(0)
seqs = torch.randint(seq // 2, seq * 3 // 2, (M,), generator=g, device=dev).to(torch.int32)
nb = (int(seqs.max()) + 15) // 16
max_blocks, n_blocks = nb + 2, M * nb + 8
tok_elems = L_s * 2 * Hkv * hd
pool = (torch.randn(n_blocks * 16 * tok_elems, device=dev) * 0.5).to(torch.bfloat16)
bt = torch.zeros(M, max_blocks, dtype=torch.int32, device=dev)
bt[:, :nb] = torch.randperm(n_blocks, device=dev)[: M * nb].view(M, nb).to(torch.int32)
q = torch.randn(M, H, hd, device=dev).to(torch.bfloat16)
out = torch.empty(M, H, hd, device=dev, dtype=torch.bfloat16)
aws = ops.AttnWorkspace(M, Hkv, hd, max_blocks, dev)
aws.set_work(seqs.cpu().numpy())
tm = ops.pool_tmap(pool, L_s, Hkv, hd)
for it in range(4):
    ops.paged_attention(tm, q, bt, seqs, out, aws, M, H, Hkv, hd, it % L_s, L_s)
torch.cuda.synchronize()
buf = np.zeros(148 * 16 * 4, dtype=np.uint64)
_C.lib().pm_attn_trace_read.argtypes = [C.c_void_p]
_C.lib().pm_attn_trace_read(buf.ctypes.data_as(C.c_void_p))
t = buf.reshape(-1, 4).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
st, fd, en, nblk = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3]
kvb = int(seqs.sum()) * 2 * Hkv * hd * 2
print(f"M={M} seq~{seq} warps={len(t)} KV {kvb/1e6:.0f} MB  span {en.max():.1f} us -> {kvb/en.max()/1e3:.0f} GB/s")
for name, v in [("start", st), ("first data", fd), ("end", en), ("blocks", nblk)]:
    q_ = np.percentile(v, [0, 10, 50, 90, 100])
    print(f"{name:10s} " + " ".join(f"{x:7.1f}" for x in q_))
hist = np.histogram(en, bins=10)
print("end-time histogram:", list(hist[0]), [f"{x:.0f}" for x in hist[1]])
busy = en - fd
live = nblk > 0
print(f"warps with work {live.sum()}/{len(t)}; us per block per warp (first data -> end): "
      f"median {np.median(busy[live] / nblk[live]):.2f}; mean warp busy {busy[live].mean():.1f} us of span {en.max():.1f}")
print(f"aggregate while streaming: {kvb / 1e3 / (en.max() - np.median(fd)):.0f} GB/s (span minus median first-data)")
