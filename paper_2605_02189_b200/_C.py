"""ctypes binding of the C-ABI library ``libpmb200.so`` (include/pm_b200.h).

There is no fallback: if the library is missing or a call fails, this module
raises.  Arguments are raw device/host pointers, sizes and a ``cudaStream_t``
(as an int); the library never allocates device memory.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PM_B200_LIB") or os.path.join(_HERE, "libpmb200.so")  # override: A/B tooling only

_P, _I, _F, _U64, _LL = C.c_void_p, C.c_int, C.c_float, C.c_ulonglong, C.c_longlong

# name -> argtypes (restype is int: a cudaError_t, 0 == success)
_SIGS = {
    "pm_abi_version": [],
    "pm_tmap_encode_2d": [_P, _P, _U64, _U64, _U64, C.c_uint, C.c_uint, _I],
    "pm_tmap_encode_pool": [_P, _P, _U64, _I, _I, _I],
    "pm_host_alloc": [_U64, C.POINTER(_P)],
    "pm_host_free": [_P],
    "pm_device_numa_node": [_I, C.POINTER(_I)],
    "pm_host_alloc_numa": [_U64, _I, C.POINTER(_P)],
    "pm_host_free_numa": [_P, _U64, _I],
    "pm_offload_rows": [_P, _P, _P, _I, _U64, _I, _P],
    "pm_host_device_ptr": [_P, C.POINTER(_P)],
    "pm_meta_upload": [_I, _P, _P, _P, _P],
    "pm_copy_pieces": [_P, _P, _P, _P, _I, _U64, _P],
    "pm_offload_gather": [_P, _P, _P, _P, _I, _U64, _P, _P, _P],
    "pm_copy_2d": [_P, _U64, _P, _U64, _U64, _U64, _P],
    "pm_gemm": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _P, _I, _P, _U64, _U64, _I, _P, _P, _I, _P],
    "pm_gemm_resid_rmsnorm": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _I, _I, _P, _U64, _U64, _P, _P, _F, _P, _I, _I, _P, _P, _I, _P],
    "pm_gemm_qkv_rope": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _I, _I, _P, _U64, _U64, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P,
                         _P, _I, _I, _I, _I, _I, _I, _F, _P],
    "pm_gemm_split_units": [_LL, _I, _I],
    "pm_gemm_split_event": [_P],
    "pm_gemm_max_segments": [_LL, _I, _I],
    "pm_gemm_fix_units": [_LL, _I, _I, _P],
    "pm_embed": [_P, _P, _P, _P, _I, _I, _P],
    "pm_rmsnorm": [_P, _P, _P, _I, _I, _F, _P],
    "pm_qkv_rope_append": [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _F, _P],
    "pm_argmax_reduce": [_P, _P, _I, _I, _I, _P, _P, _P, _P],
    "pm_paged_attention": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P],
    "pm_attn_work_list": [_P, _I, _I, _I, _I, _I, _I, _P],
    "pm_attn_workers": [_I],
    "pm_attn_workers_cfg": [_I, _I],
    "pm_attn_max_piece": [],
    "pm_prepare_gemm": [],
    "pm_prepare_attention": [],
    "pm_hop_pack": [_P, _P, _LL, _P],
    "pm_hop_unpack": [_P, _P, _LL, _P],
    "pm_scatter_tokens": [_P, _P, _I, _P, _P],
    "pm_gemm_cl": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I, _P, _I, _I, _F, _P, _P, _P, _P, _P, _P,
                   _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P],
    "pm_gemm_cl_max_clusters": [_I, _I, C.POINTER(_I)],
    "pm_gemm_cl_stages": [_I],
    "pm_gemm_cl_trace_read": [_P],
    "pm_prepare_gemm_cl": [],
}

_lib = None


class KernelError(RuntimeError):
    pass


def lib():
    """Load the library once; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing -- run __graft_entry__.build() (no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, argt in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = argt
            fn.restype = _I
        handle.pm_error_string.argtypes = [_I]
        handle.pm_error_string.restype = C.c_char_p
        _lib = handle
    return _lib


def call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().pm_error_string(rc).decode()
        raise KernelError(f"{name} failed: cudaError {rc} ({msg})")
    return rc


def exported_symbols():
    return sorted(_SIGS) + ["pm_error_string"]
