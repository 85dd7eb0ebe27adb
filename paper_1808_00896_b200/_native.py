"""ctypes binding of the C ABI in include/so3fft_b200.h (libso3fft_b200.so, built in-tree).

There is no CPU fallback: if the shared library is missing, importing the
transforms raises ``NativeLibraryError``.  Status codes map to the reference's
exception types: SO3_ERR_INVALID -> ValueError (as the reference's argument
checks, e.g. soft.py:118-121, core.py:34-40), anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libso3fft_b200.so")

SO3_OK = 0
SO3_ERR_INVALID = 1
SO3_ERR_CUDA = 2
SO3_ERR_NOMEM = 3

_c_int, _c_i64, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)

# name -> (restype, argtypes); the full export list of include/so3fft_b200.h
SIGNATURES = {
    "so3_last_error": (ctypes.c_char_p, []),
    "so3_version": (ctypes.c_char_p, []),
    "so3_coeff_count": (_c_i64, [_c_int]),
    "so3_grid_count": (_c_i64, [_c_int]),
    "so3_coeff_index": (_c_i64, [_c_int, _c_int, _c_int, _c_int]),
    "so3_quadrature_weights": (_c_int, [_c_int, _dp]),
    "so3_sample_angles": (_c_int, [_c_int, _dp, _dp]),
    "so3_cluster_count": (_c_i64, [_c_int]),
    "so3_cluster_schedule": (_c_int, [_c_int, _i32p, _i32p]),
    "so3_plan_create": (_c_int, [_c_int, _c_int, ctypes.POINTER(_vp)]),
    "so3_plan_destroy": (None, [_vp]),
    "so3_plan_bandwidth": (_c_int, [_vp]),
    "so3_plan_batch": (_c_int, [_vp]),
    "so3_plan_device": (_c_int, [_vp]),
    "so3_plan_device_bytes": (_c_i64, [_vp]),
    "so3_fsoft": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_ifsoft": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_fsoft_host": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_ifsoft_host": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_fft_analysis": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_fft_synthesis": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_dwt_analysis": (_c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _vp]),
    "so3_dwt_synthesis": (_c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _vp]),
    "so3_plan_scratch": (_vp, [_vp]),
    "so3_plan_set_dwt_variant": (_c_int, [_vp, _c_int]),
    "so3_plan_set_knob": (_c_int, [_vp, ctypes.c_char_p, _c_int]),
    "so3_wigner_rows": (_c_int, [_vp, _c_int, _c_int, _vp, _vp]),
    "so3_container_info": (_c_int, [ctypes.c_char_p, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int),
                                    ctypes.POINTER(_c_i64)]),
    "so3_read_container": (_c_int, [ctypes.c_char_p, _c_int, _c_int, _c_int, _vp, _c_int, _c_i64, _vp]),
    "so3_write_container": (_c_int, [ctypes.c_char_p, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _c_i64,
                                     _vp]),
    "so3_jacobi_eval": (_c_int, [_c_int, ctypes.c_double, ctypes.c_double, _vp, _c_i64, _vp, _vp]),
    "so3_wigner_d_eval": (_c_int, [_c_int, _c_int, _c_int, _vp, _c_i64, _vp, _vp]),
    "so3_wigner_rows_eval": (_c_int, [_c_int, _c_int, _c_int, _vp, _c_i64, _vp, _vp]),
    "so3_fsoft_direct": (_c_int, [_c_int, _vp, _vp, _vp]),
    "so3_ifsoft_direct": (_c_int, [_c_int, _vp, _vp, _vp]),
    "so3_shard_plan_create": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(_vp)]),
    "so3_shard_plan_create_chunked": (_c_int, [_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_vp)]),
    "so3_shard_chunks": (_c_i64, [_vp]),
    "so3_shard_chunk_pairs": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(_c_i64)]),
    "so3_shard_dwt_analysis_chunk": (_c_int, [_vp, _c_int, _vp, _vp, _vp]),
    "so3_shard_dwt_synthesis_chunk": (_c_int, [_vp, _c_int, _vp, _vp, _vp]),
    "so3_shard_slab_width": (_c_i64, [_vp]),
    "so3_shard_rank_pairs": (_c_i64, [_vp]),
    "so3_shard_pair_counts": (_c_int, [_c_int, _c_int, ctypes.POINTER(_c_i64)]),
    "so3_shard_cluster_owner": (_c_int, [_c_int, _c_int, _i32p]),
    "so3_shard_pair_list": (_c_int, [_c_int, _c_int, _c_int, _i32p]),
    "so3_shard_fft_analysis": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_shard_dwt_analysis": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_shard_dwt_synthesis": (_c_int, [_vp, _vp, _vp, _vp]),
    "so3_shard_fft_synthesis": (_c_int, [_vp, _vp, _vp, _vp]),
}


class NativeLibraryError(ImportError):
    """The CUDA library is not built or cannot be loaded (no fallback exists)."""


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libso3fft_b200.so once and attach the C signatures."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return _lib


def check(status: int, what: str) -> None:
    """Raise the reference-equivalent exception for a nonzero status."""
    if status == SO3_OK:
        return
    msg = lib().so3_last_error().decode(errors="replace")
    if status == SO3_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    if status == SO3_ERR_NOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")
