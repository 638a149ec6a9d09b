"""CPU-side checks of the C-ABI library and the host logic around it: the
library loads and exports every symbol include/pm_b200.h declares; the
weight packing reproduces the UMMA 128B-swizzle image; the stream-K
partition (mirrored in Python) covers every k-block exactly once and the
library's segment count matches."""
import os
import re

import pytest
import torch

from paper_2605_02189_b200 import _C, ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    lib = _C.lib()
    hdr = open(os.path.join(ROOT, "include", "pm_b200.h")).read()
    names = re.findall(r"\b(pm_[a-z0-9_]+)\s*\(", hdr)
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(_C.exported_symbols())
    assert lib.pm_abi_version() == 1


def test_pack_weight_swizzle_image():
    n, k = 300, 192
    w = torch.randn(n, k).to(torch.bfloat16)
    packed, units = ops.pack_weight(w)
    assert units == 2 and packed.shape == (2, 3, 2, 128, 8, 8)
    flat = packed.reshape(units, 3, 2, 128, 64)
    for (u, kb, h, r, c) in [(0, 0, 0, 0, 0), (0, 1, 1, 5, 3), (1, 2, 0, 43, 7), (0, 2, 1, 127, 1), (1, 0, 1, 100, 2)]:
        row = u * 256 + h * 128 + r
        chunk = c ^ (r % 8)
        got = flat[u, kb, h, r, chunk * 8:(chunk + 1) * 8]
        want = w[row, kb * 64 + c * 8: kb * 64 + c * 8 + 8] if row < n else torch.zeros(8, dtype=w.dtype)
        assert torch.equal(got, want)


def _owner(idx, T, G):
    return ((idx + 1) * G + T - 1) // T - 1


@pytest.mark.parametrize("units,kb,grid", [(24, 64, 148), (16, 64, 148), (594, 64, 148), (2, 4, 8), (1, 1, 2),
                                           (96, 64, 148), (20, 400, 148)])
def test_stream_k_partition(units, kb, grid):
    T = units * kb
    G = min(grid // 2, T)   # stream-K workers are CTA pairs
    seen = [0] * T
    for c in range(G):
        lo, hi = c * T // G, (c + 1) * T // G
        for i in range(lo, hi):
            seen[i] += 1
            assert _owner(i, T, G) == c
    assert all(x == 1 for x in seen)
    segs = max(_owner((u + 1) * kb - 1, T, G) - _owner(u * kb, T, G) + 1 for u in range(units))
    assert _C.lib().pm_gemm_max_segments(T, kb, G) == segs


@pytest.mark.parametrize("lens,hkv,workers", [([1, 17, 300, 129, 128], 2, 4), ([5], 8, 1776),
                                               ([1000, 2, 77, 513], 1, 3), ([16] * 9, 2, 6),
                                               (list(range(1, 400, 7)), 8, 64)])
def test_attention_work_list_host_helpers_agree(lens, hkv, workers):
    """The C helper (what a non-Python host would call) and the numpy one the
    engine uses build the same balanced piece list (tests/test_attn_work_list.py
    checks its coverage and balance at the bench shapes)."""
    import numpy as np
    seq = np.asarray(lens, dtype=np.int32)
    cap = ops.attn_work_len(len(lens), hkv, max(-(-L // 16) for L in lens), workers)
    buf = np.zeros(cap, dtype=np.int32)
    n = _C.lib().pm_attn_work_list(seq.ctypes.data_as(_C.C.c_void_p), len(lens), hkv, workers, ops.ATTN_MAXP,
                                   ops.ATTN_MINQ, cap, buf.ctypes.data_as(_C.C.c_void_p))
    ref = ops.attn_work_list(seq, hkv, workers)
    assert n == len(ref) == ops.attn_work_used(ref)
    assert np.array_equal(buf[:n], ref)
