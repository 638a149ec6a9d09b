"""Host logic of the balanced attention work split (ops.attn_work_list, the
C mirror pm_attn_work_list): every (row, kv head)'s KV blocks covered exactly
once, in order, by pieces of at most ATTN_MAXP blocks; every warp gets the
same number of blocks (the quota q; the last warp the remainder); a piece's
chunk / nchunks are its rank / count within its (row, head) -- the merge
order.  Runs on CPU (the C builder is host code in libpmb200.so)."""
import ctypes

import numpy as np
import pytest

from paper_2605_02189_b200 import _C, ops

CASES = [
    ("C2 qwen3-8b 121 rows", 8, 1776, np.random.default_rng(0).integers(512, 1025, 121)),
    ("C3 stage 48 rows", 8, 1184, np.random.default_rng(1).integers(1000, 1100, 48)),
    ("C4 stage 24 rows", 8, 1776, np.random.default_rng(2).integers(1000, 1100, 24)),
    ("C5 256 rows", 8, 1184, np.random.default_rng(3).integers(1024, 1100, 256)),
    ("tiny / ragged", 2, 1776, np.array([1, 17, 40, 0, 300, 5])),
    ("one row", 8, 1776, np.array([2049])),
    ("prefill chunk (causal rows)", 8, 1184, np.arange(100, 164) + 1),
]


def decode(w):
    used, P = int(w[0]), int(w[1])
    off = w[2:3 + used].astype(np.int64)
    base = (3 + used + 3) // 4 * 4
    pc = w[base:base + 4 * P].reshape(P, 4).astype(np.int64)
    row, kvh = pc[:, 0] & 0xffff, pc[:, 0] >> 16
    b0, nblk = pc[:, 1] & 0xffff, pc[:, 1] >> 16
    chunk, nchunks = pc[:, 2] & 0xffff, pc[:, 2] >> 16
    return used, off, row, kvh, b0, nblk, chunk, nchunks, pc[:, 3]


@pytest.mark.parametrize("name,hkv,workers,seq", CASES, ids=[c[0] for c in CASES])
def test_balanced_work_list(name, hkv, workers, seq):
    w = ops.attn_work_list(seq, hkv, workers)
    used, off, row, kvh, b0, nblk, chunk, nchunks, s = decode(w)
    nb = (seq + 15) // 16
    B = int(nb.sum()) * hkv
    q = max(ops.ATTN_MINQ, -(-B // workers))
    assert used == -(-B // q) <= workers
    assert (nblk >= 1).all() and (nblk <= ops.ATTN_MAXP).all()
    assert (s == seq[row]).all()
    # exact, ordered coverage of every (row, head)'s blocks
    for r in range(len(seq)):
        for h in range(hkv):
            sel = np.nonzero((row == r) & (kvh == h))[0]
            if nb[r] == 0:
                assert len(sel) == 0
                continue
            assert (b0[sel] == np.concatenate([[0], np.cumsum(nblk[sel])[:-1]])).all()
            assert nblk[sel].sum() == nb[r]
            assert (chunk[sel] == np.arange(len(sel))).all() and (nchunks[sel] == len(sel)).all()
    # every warp streams q blocks (the last one the rest)
    per_warp = np.array([nblk[off[i]:off[i + 1]].sum() for i in range(used)])
    assert (per_warp[:-1] == q).all() and 0 < per_warp[-1] <= q
    assert ops.attn_work_used(w) == len(w)
    # pieces of one (row, head) bounded by the workspace's max_chunks
    assert nchunks.max() <= ops.attn_max_chunks(int(nb.max()))


@pytest.mark.parametrize("name,hkv,workers,seq", CASES, ids=[c[0] for c in CASES])
def test_c_builder_matches_numpy(name, hkv, workers, seq):
    want = ops.attn_work_list(seq, hkv, workers)
    cap = ops.attn_work_len(len(seq), hkv, int(((seq + 15) // 16).max()), workers)
    got = np.zeros(cap, dtype=np.int32)
    s32 = np.ascontiguousarray(seq, dtype=np.int32)
    lib = _C.lib()
    lib.pm_attn_work_list.restype = ctypes.c_int
    n = lib.pm_attn_work_list(s32.ctypes.data_as(ctypes.c_void_p), len(seq), hkv, workers, ops.ATTN_MAXP,
                              ops.ATTN_MINQ, cap, got.ctypes.data_as(ctypes.c_void_p))
    assert n == len(want)
    assert np.array_equal(got[:n], want)
    assert lib.pm_attn_max_piece() == ops.ATTN_MAXP


def test_work_len_bound_holds():
    rng = np.random.default_rng(9)
    for _ in range(50):
        m = int(rng.integers(1, 300))
        mb = int(rng.integers(1, 130))
        seq = rng.integers(0, mb * 16 + 1, m)
        workers = int(rng.choice([592, 1184, 1776]))
        w = ops.attn_work_list(seq, 8, workers)
        assert ops.attn_work_used(w) <= ops.attn_work_len(m, 8, mb, workers)


def test_engine_passes_rows_per_step():
    from paper_2605_02189_b200.engine import attn_rows_hint
    assert attn_rows_hint(512, 8) == 64 and attn_rows_hint(256, 2) == 128 and attn_rows_hint(256, 8) == 32
    assert attn_rows_hint(10, 3) == 4
