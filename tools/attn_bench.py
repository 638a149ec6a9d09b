"""Time paged attention alone on decode shapes (CUDA events; pool >> L2)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_02189_b200 import ops  # noqa: E402
from paper_2605_02189_b200.models import QWEN3_8B, QWEN3_32B  # noqa: E402

dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
for spec, L_s, M, seq, rag in [(QWEN3_8B, 36, 128, 550, 0), (QWEN3_8B, 36, 128, 550, 1), (QWEN3_8B, 36, 128, 1000, 1),
                               (QWEN3_32B, 8, 64, 1024, 0), (QWEN3_32B, 16, 256, 300, 1), (QWEN3_8B, 36, 16, 2000, 1)]:
    H, Hkv, hd = spec.H, spec.Hkv, spec.hd
    if rag:  # ragged lengths in [seq/2, 3seq/2]
        seqs_l = torch.randint(seq // 2, seq * 3 // 2, (M,), generator=g, device=dev)
    else:
        seqs_l = torch.full((M,), seq, device=dev)
    nb = (int(seqs_l.max()) + 15) // 16
    max_blocks = nb + 2
    n_blocks = M * nb + 8
    tok_elems = L_s * 2 * Hkv * hd
    pool = (torch.randn(n_blocks * 16 * tok_elems, device=dev) * 0.5).to(torch.bfloat16)
    perm = torch.randperm(n_blocks, device=dev)[: M * nb].view(M, nb).to(torch.int32)
    bt = torch.zeros(M, max_blocks, dtype=torch.int32, device=dev)
    bt[:, :nb] = perm
    seqs = seqs_l.to(torch.int32)
    q = torch.randn(M, H, hd, device=dev).to(torch.bfloat16)
    out = torch.empty(M, H, hd, device=dev, dtype=torch.bfloat16)
    aws = ops.AttnWorkspace(M, Hkv, hd, max_blocks, dev)
    tm = ops.pool_tmap(pool, L_s, Hkv, hd)
    aws.set_work(seqs.cpu().numpy())
    ts = []
    for it in range(12):
        layer = it % L_s
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.paged_attention(tm, q, bt, seqs, out, aws, M, H, Hkv, hd, layer, L_s)
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b) * 1e-3)
    t = min(ts)
    kvb = int(seqs.sum()) * 2 * Hkv * hd * 2
    print(f"{spec.name} L_s={L_s} M={M} seq={seq} ragged={rag}: {t*1e6:7.1f} us  {kvb/t/1e9:6.0f} GB/s")
    del pool
