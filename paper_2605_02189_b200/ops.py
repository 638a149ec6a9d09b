"""Tensor-level wrappers over the C-ABI kernels (torch for device memory and
streams only).  Every op runs a hand-written sm_100a kernel from
``libpmb200.so``; there is no eager/PyTorch fallback."""

from __future__ import annotations

import ctypes as C
import math

import torch

from . import _C

SMS = 148
BM, BK = 128, 64


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class TensorMap:
    """A 64-byte-aligned host copy of a CUtensorMap (passed by value to the
    kernels).  Keeps the described tensor alive."""

    def __init__(self, tensor, inner, outer, row_stride_bytes, box_inner, box_outer, swizzle=True):
        self._raw = (C.c_ubyte * 192)()
        addr = C.addressof(self._raw)
        self.addr = (addr + 63) & ~63
        self.tensor = tensor
        _C.call("pm_tmap_encode_2d", C.c_void_p(self.addr), C.c_void_p(tensor.data_ptr()),
                inner, outer, row_stride_bytes, box_inner, box_outer, 1 if swizzle else 0)

    @property
    def ptr(self):
        return C.c_void_p(self.addr)


def matrix_tmap(t: torch.Tensor, box_rows: int) -> TensorMap:
    """K-major bf16 matrix [rows, K] -> TMA map with a [box_rows x 64] box."""
    assert t.dtype == torch.bfloat16 and t.dim() == 2 and t.stride(1) == 1
    return TensorMap(t, t.shape[1], t.shape[0], t.stride(0) * 2, BK, box_rows)


def choose_splits(n_out: int, k: int, sms: int = SMS) -> int:
    """Fixed K-split of a projection, a function of its shape only (never of
    the micro-batch size) so results are batch-invariant.  Minimises
    waves x (k-blocks per CTA + fixed per-CTA overhead)."""
    tiles, kb = n_out // BM, k // BK
    best = (math.inf, 1)
    for s in range(1, min(16, max(1, kb // 4)) + 1):
        cost = math.ceil(tiles * s / sms) * (kb / s + 6.0)
        if cost < best[0] - 1e-9:
            best = (cost, s)
    return best[1]


def bn_for(m_tok: int) -> int:
    for bn in (16, 32, 64, 128, 256):
        if m_tok <= bn:
            return bn
    return 256


EPI_STORE_BF16, EPI_RESID_ADD, EPI_SILU_MUL, EPI_LOGITS_ARGMAX = 0, 1, 2, 3


class GemmWorkspace:
    """Split-K partials, per-tile counters and argmax partials shared by all
    projections of one executor (ops on one stream run in order)."""

    def __init__(self, m_cap: int, max_n_out: int, max_splits: int, vocab_tiles: int, device):
        self.m_cap = m_cap
        self.ws = torch.empty(max_splits * m_cap * max_n_out, dtype=torch.float32, device=device)
        tok_tiles = max(1, math.ceil(m_cap / 256))
        self.counters = torch.zeros(tok_tiles * max(vocab_tiles, max_n_out // BM), dtype=torch.int32, device=device)
        self.amax_val = torch.empty(max(1, vocab_tiles) * m_cap, dtype=torch.float32, device=device)
        self.amax_idx = torch.empty(max(1, vocab_tiles) * m_cap, dtype=torch.int32, device=device)


class Linear:
    """One projection: weight [n_out, K] bf16 (K-major) + its TMA map + fixed split."""

    def __init__(self, weight: torch.Tensor, splits: int = None):
        assert weight.is_contiguous() and weight.dtype == torch.bfloat16
        self.w = weight
        self.n_out, self.k = weight.shape
        assert self.n_out % BM == 0 and self.k % BK == 0, (self.n_out, self.k)
        self.tmap = matrix_tmap(weight, BM)
        self.splits = splits or choose_splits(self.n_out, self.k)

    def __call__(self, x_maps: dict, m_tok: int, epilogue: int, out, ld_out: int, ws: GemmWorkspace,
                 stream=None, splits: int = None):
        bn = bn_for(m_tok)
        s = splits or self.splits
        if epilogue == EPI_LOGITS_ARGMAX:
            s = 1
        _C.call("pm_gemm", self.tmap.ptr, x_maps[bn].ptr, self.n_out, self.k, m_tok, bn, s, epilogue,
                _ptr(out), ld_out, _ptr(ws.ws), ws.m_cap, _ptr(ws.counters), _ptr(ws.amax_val),
                _ptr(ws.amax_idx), _stream(stream))


def activation_maps(buf: torch.Tensor) -> dict:
    """TMA maps of an activation buffer [m_cap, K] for every supported BN."""
    return {bn: matrix_tmap(buf, bn) for bn in (16, 32, 64, 128, 256)}


def embed(tok_table, slots, table, resid, M, stream=None):
    _C.call("pm_embed", _ptr(tok_table), _ptr(slots), _ptr(table), _ptr(resid), M, table.shape[1], _stream(stream))


def rmsnorm(x, w, y, M, eps, stream=None):
    _C.call("pm_rmsnorm", _ptr(x), _ptr(w), _ptr(y), M, x.shape[-1], eps, _stream(stream))


def qkv_rope_append(qkv, q_out, pool, block_table, positions, rope, qn_w, kn_w, M, H, Hkv, hd, layer,
                    L_s, eps, stream=None):
    _C.call("pm_qkv_rope_append", _ptr(qkv), _ptr(q_out), _ptr(pool), _ptr(block_table), _ptr(positions),
            _ptr(rope), _ptr(qn_w), _ptr(kn_w), M, H, Hkv, hd, layer, L_s, block_table.shape[1], eps,
            _stream(stream))


def pool_tmap(pool: torch.Tensor, L_s: int, Hkv: int, hd: int) -> TensorMap:
    """2-D TMA view of the block-first pool: rows = block*16 + slot, cols =
    (layer, k|v, head, dim); box = 16 slots x 64 dims, 128B swizzle."""
    n_rows = pool.numel() // (L_s * 2 * Hkv * hd)
    width = L_s * 2 * Hkv * hd
    return TensorMap(pool, width, n_rows, width * 2, 64, 16)


def attn_blocks_per_split() -> int:
    return _C.lib().pm_attn_blocks_per_split()


def paged_attention(tmap_kv, q, block_table, seq_lens, out, ws_o, ws_ml, counters, M, H, Hkv, hd, layer,
                    L_s, max_splits, stream=None):
    _C.call("pm_paged_attention", tmap_kv.ptr, _ptr(q), _ptr(block_table), _ptr(seq_lens), _ptr(out),
            _ptr(ws_o), _ptr(ws_ml), _ptr(counters), M, H, Hkv, hd, layer, L_s, block_table.shape[1],
            max_splits, _stream(stream))


def argmax_reduce(ws: GemmWorkspace, n_tiles, M, out_ids, tok_table=None, slots=None, stream=None):
    _C.call("pm_argmax_reduce", _ptr(ws.amax_val), _ptr(ws.amax_idx), n_tiles, M, ws.m_cap, _ptr(out_ids),
            _ptr(tok_table), _ptr(slots), _stream(stream))
