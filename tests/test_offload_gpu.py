"""Decode offload paths (kv.OFFLOAD_MODE): the gathered single-DMA offload
(pm_offload_gather: gather kernel -> one cudaMemcpyAsync -> host scatter in
stream order) and the per-row DMAs (pm_copy_pieces) leave the pinned host
replica a bit-exact copy of the KV in HBM -- directly on random rows, and
through the engine across evict / prefetch round trips (a prefetch that
reads a replica slot is ordered after the offload that wrote it)."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2605_02189_b200 import _C, kv

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bytes_", [(1, 4096), (37, 32768), (121, 147456), (2500, 1024)])
def test_offload_gather_places_rows(n, bytes_):
    rng = np.random.default_rng(n)
    n_slots = n + 7
    pool = torch.randint(0, 255, (n_slots * bytes_,), dtype=torch.uint8, device="cuda")
    pool_off = (rng.permutation(n_slots)[:n] * bytes_).astype(np.int64)
    rep_bytes = (n + 3) * bytes_ * 2
    rep_p = _C.C.c_void_p()
    _C.call("pm_host_alloc", rep_bytes, _C.C.byref(rep_p))
    host_p = _C.C.c_void_p()
    _C.call("pm_host_alloc", n * bytes_, _C.C.byref(host_p))
    try:
        rep = np.frombuffer((ctypes.c_uint8 * rep_bytes).from_address(rep_p.value), dtype=np.uint8)
        rep[:] = 0
        rep_off = (rng.permutation(2 * (n + 3))[:n] * bytes_).astype(np.int64)
        stage = torch.empty(n * bytes_, dtype=torch.uint8, device="cuda")
        st = torch.cuda.Stream()
        _C.call("pm_offload_gather", rep_p, _C.C.c_void_p(pool.data_ptr()), rep_off.ctypes.data_as(_C.C.c_void_p),
                pool_off.ctypes.data_as(_C.C.c_void_p), n, bytes_, _C.C.c_void_p(stage.data_ptr()), host_p,
                _C.C.c_void_p(st.cuda_stream))
        st.synchronize()   # the host scatter ran in stream order before this returns
        p = pool.cpu().numpy()
        for i in range(n):
            assert np.array_equal(rep[rep_off[i]:rep_off[i] + bytes_], p[pool_off[i]:pool_off[i] + bytes_]), i
    finally:
        _C.call("pm_host_free", rep_p)
        _C.call("pm_host_free", host_p)


@pytest.mark.parametrize("mode", ["gather", "dma"])
def test_engine_replica_bit_exact_per_offload_mode(mode, monkeypatch):
    from test_engine_gpu import build, check_replica
    monkeypatch.setattr(kv, "OFFLOAD_MODE", mode)
    spec, eng, reqs, prompts = build(n_req=24, m=4, cap=40, seed=7)
    n = 0
    while n < 40 and eng.step() is not None:
        n += 1
    assert eng.n_evicted > 0 and eng.n_prefetched > 0
    check_replica(eng)


def test_chunk_pinned_replica_copies_across_pieces():
    """The replica is pinned in 1 GB pieces (pm_host_alloc_numa): copies that
    straddle a piece boundary still move the right bytes, both directions."""
    from paper_2605_02189_b200.kv import device_numa_node
    nbytes = (2 << 30) + (64 << 20)
    node = max(0, device_numa_node())
    p = _C.C.c_void_p()
    _C.call("pm_host_alloc_numa", nbytes, node, _C.C.byref(p))
    try:
        host = np.frombuffer((ctypes.c_uint8 * nbytes).from_address(p.value), dtype=np.uint8)
        lo, n = (1 << 30) - (3 << 20), 6 << 20          # 3 MB each side of the first boundary
        host[lo:lo + n] = np.random.default_rng(1).integers(0, 255, n, dtype=np.uint8)
        dev = torch.empty(n, dtype=torch.uint8, device="cuda")
        st = torch.cuda.Stream()
        off = np.array([0], dtype=np.int64)
        src = np.array([lo], dtype=np.int64)
        _C.call("pm_copy_pieces", _C.C.c_void_p(dev.data_ptr()), p, off.ctypes.data_as(_C.C.c_void_p),
                src.ctypes.data_as(_C.C.c_void_p), 1, n, _C.C.c_void_p(st.cuda_stream))
        st.synchronize()
        assert np.array_equal(dev.cpu().numpy(), host[lo:lo + n])
        dev.add_(1)
        dst = np.array([lo + (1 << 30)], dtype=np.int64)   # straddles the second boundary
        _C.call("pm_copy_pieces", p, _C.C.c_void_p(dev.data_ptr()), dst.ctypes.data_as(_C.C.c_void_p),
                off.ctypes.data_as(_C.C.c_void_p), 1, n, _C.C.c_void_p(st.cuda_stream))
        st.synchronize()
        assert np.array_equal(host[lo + (1 << 30):lo + (1 << 30) + n], dev.cpu().numpy())
    finally:
        _C.call("pm_host_free_numa", p, nbytes, node)
