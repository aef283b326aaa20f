"""ctypes binding of librgb200.so (include/rgb200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every device entry point raises instead of silently
computing on the host.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

_PKG = pathlib.Path(__file__).resolve().parent
# RG_LIB_PATH selects an alternative build of the same library (tools/ab_build.py variants)
LIB_PATH = pathlib.Path(os.environ["RG_LIB_PATH"]) if os.environ.get("RG_LIB_PATH") else _PKG / "_lib" / "librgb200.so"

RG_OK, RG_EBADARG, RG_ECUDA = 0, 1, 2

c_i32, c_i64, c_dbl, c_ptr = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/rgb200.h
PROTOTYPES = {
    "rg_version": (ctypes.c_char_p, []),
    "rg_last_error": (ctypes.c_char_p, []),
    "rg_device_sm_count": (ctypes.c_int, []),
    "rg_spmm_csr_f64": (ctypes.c_int, [c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64,
                                       c_ptr, c_i64, c_i32, c_ptr, c_i64, c_ptr]),
    "rg_tall_f64": (ctypes.c_int, [c_i64, c_i32, c_ptr, c_i64, c_ptr, c_i64,
                                   c_ptr, c_i64, c_i32, c_ptr, c_dbl,
                                   c_ptr, c_i64, c_i32, c_ptr, c_dbl,
                                   c_ptr, c_ptr, c_i32, c_ptr, c_i64, c_i32, c_ptr,
                                   c_ptr, c_i64, c_ptr]),
    "rg_tall_workspace_bytes": (c_i64, [c_i64, c_i32, c_i32, c_i32, c_i32, c_i32]),
    "rg_chol_f64": (ctypes.c_int, [c_i32, c_ptr, c_ptr, c_ptr, c_dbl, c_ptr]),
    "rg_tsqr_f64": (ctypes.c_int, [c_i64, c_i32, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr]),
    "rg_tsqr_workspace_bytes": (c_i64, [c_i64, c_i32]),
    "rg_cgs2_f64": (ctypes.c_int, [c_i64, c_i32, c_ptr, c_i64, c_ptr, c_i64, c_i32, c_ptr, c_i64, c_i32,
                                   c_ptr, c_ptr, c_i32, c_ptr, c_i64, c_ptr]),
    "rg_cholqr2_f64": (ctypes.c_int, [c_i64, c_i32, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr, c_i32,
                                      c_ptr, c_i64, c_ptr]),
    "rg_spmm_csr_c128": (ctypes.c_int, [c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64,
                                        c_ptr, c_i64, c_i32, c_ptr, c_i64, c_ptr]),
    "rg_tall_c128": (ctypes.c_int, [c_i64, c_i32, c_ptr, c_i64, c_ptr, c_i64,
                                    c_ptr, c_i64, c_i32, c_ptr, c_dbl,
                                    c_ptr, c_i64, c_i32, c_ptr, c_dbl,
                                    c_ptr, c_ptr, c_i32, c_ptr, c_i64, c_i32, c_ptr,
                                    c_ptr, c_i64, c_ptr]),
    "rg_tall_c128_workspace_bytes": (c_i64, [c_i64, c_i32, c_i32, c_i32, c_i32, c_i32]),
    "rg_chol_c128": (ctypes.c_int, [c_i32, c_ptr, c_ptr, c_ptr, c_dbl, c_ptr]),
    "rg_wave_workspace_bytes": (c_i64, [c_i64]),
    "rg_wave_max_chunks": (c_i64, [c_i64]),
    "rg_wave_schedule": (c_i32, [c_i64, c_ptr, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr]),
    "rg_ilu0_f64": (ctypes.c_int, [c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr,
                                   c_i64, c_i32, c_ptr]),
    "rg_wave_permute": (c_i64, [c_i64, c_ptr, c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "rg_gather_f64": (ctypes.c_int, [c_i64, c_ptr, c_ptr, c_ptr, c_ptr]),
    "rg_spmm_dia_f64": (ctypes.c_int, [c_i64, c_i64, c_i64, c_i32, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_i64,
                                       c_i32, c_ptr, c_i64, c_ptr, c_ptr]),
    "rg_dia_offsets": (ctypes.c_int, [c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr]),
    "rg_dia_fill_f64": (ctypes.c_int, [c_i64, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_i64, c_ptr,
                                       c_ptr]),
    "rg_halo_pack": (ctypes.c_int, [c_i64, c_i32, c_i32, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr]),
    "rg_permute_rows_f64": (ctypes.c_int, [c_i64, c_i32, c_ptr, c_i64, c_ptr, c_ptr, c_i64, c_ptr, c_ptr]),
    "rg_sptrsv_perm_f64": (ctypes.c_int, [c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i32, c_i32, c_i32, c_ptr,
                                          c_ptr, c_i64, c_i32, c_ptr]),
    "rg_sptrsv_f64": (ctypes.c_int, [c_i64, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr, c_i32, c_i32, c_i32, c_i32,
                                     c_ptr,
                                     c_i64, c_ptr, c_i64, c_ptr, c_i64, c_i32, c_ptr]),
    "rg_halo_push": (ctypes.c_int, [c_i64, c_i32, c_i32, c_ptr, c_ptr, c_i64, c_ptr, c_i64, c_ptr, ctypes.c_uint32,
                                    c_ptr, c_ptr]),
    "rg_halo_wait": (ctypes.c_int, [c_ptr, ctypes.POINTER(c_i32), c_i32, ctypes.c_uint32, c_dbl, c_ptr, c_ptr]),
    "rg_ipc_alloc": (ctypes.c_int, [c_i64, ctypes.POINTER(c_ptr), c_ptr]),
    "rg_peer_buffer_bytes": (c_i64, []),
    "rg_peer_alloc": (ctypes.c_int, [ctypes.POINTER(c_ptr), c_ptr]),
    "rg_peer_open": (ctypes.c_int, [c_ptr, ctypes.POINTER(c_ptr)]),
    "rg_peer_close": (ctypes.c_int, [c_ptr]),
    "rg_peer_free": (ctypes.c_int, [c_ptr]),
    "rg_peer_set": (ctypes.c_int, [c_i32, c_i32, ctypes.POINTER(c_ptr), c_dbl]),
    "rg_peer_clear": (None, []),
    "rg_peer_active": (c_i32, []),
    "rg_peer_error": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32), c_ptr]),
    "rg_peer_allreduce_f64": (ctypes.c_int, [c_ptr, c_i64, c_ptr]),
    "rg_peer_emulate_f64": (ctypes.c_int, [c_i32, c_i32, c_i32, ctypes.c_uint32, c_ptr, c_ptr, c_ptr]),
    "rg_launch_count": (c_i64, []),
    "rg_count_launches": (None, [c_i64]),
    "rg_profile_enable": (None, [c_i32]),
    "rg_profile_count": (c_i32, []),
    "rg_profile_record": (ctypes.c_int, [c_i32, ctypes.c_char_p, c_i32, ctypes.POINTER(c_dbl),
                                         ctypes.POINTER(c_i64), ctypes.POINTER(c_dbl), ctypes.POINTER(c_i32)]),
    "rg_profile_gap": (ctypes.c_int, [c_i32, ctypes.POINTER(c_dbl)]),
}

_lib = None
_lock = threading.Lock()


class KernelError(RuntimeError):
    """A CUDA launch inside librgb200 failed."""


def load(required_symbols=None):
    """Load librgb200.so (building it first if it is absent and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            from . import build as _build

            _build.build()
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols():
    lib = load()
    return sorted(n for n in PROTOTYPES if getattr(lib, n, None) is not None)


def check(rc: int, what: str):
    """Map an rg_* status to the reference's exception classes."""
    if rc == RG_OK:
        return
    msg = (_lib.rg_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    if rc == RG_EBADARG:
        from .sparse_core import ShapeError

        raise ShapeError(f"{what}: {msg}")
    raise KernelError(f"{what}: {msg}")
