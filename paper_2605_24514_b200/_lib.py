"""ctypes binding of libisvd.so (the C ABI declared in include/isvd.h).

There is deliberately no fallback: if the shared library is missing or no
CUDA device is present, every engine call raises.  The library is built
in-tree by ``paper_2605_24514_b200.build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libisvd.so"

ISVD_OK = 0
ISVD_EINVAL = 1
ISVD_ENODEV = 2
ISVD_ENOMEM = 3
ISVD_ESTATE = 4

_dp = C.POINTER(C.c_double)
_ip64 = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol include/isvd.h declares.
SIGNATURES = {
    "isvd_last_error": (C.c_char_p, []),
    "isvd_version": (C.c_int, []),
    "isvd_launch_count": (C.c_int64, []),
    "isvd_debug_counters": (C.c_int, [_ip64, C.c_int]),
    "isvd_debug_trace": (C.c_int, [_ip64, C.c_int]),
    "isvd_core_svd": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "isvd_row_append": (C.c_int, [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_double,
                                  C.c_int, _dp, _dp, _dp, _dp]),
    "isvd_rank_one": (C.c_int, [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int64, C.c_int64,
                                C.c_double, C.c_int, _dp, _dp, _dp]),
    "isvd_engine_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _vp]),
    "isvd_engine_destroy": (C.c_int, [_vp]),
    "isvd_engine_init": (C.c_int, [_vp, _vp, C.c_int]),
    "isvd_engine_row_append": (C.c_int, [_vp, _vp, C.c_int]),
    "isvd_engine_col_append": (C.c_int, [_vp, _vp, C.c_int]),
    "isvd_engine_rank_one": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int]),
    "isvd_engine_refresh": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_set_reference": (C.c_int, [_vp]),
    "isvd_engine_set_rank": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_shape": (C.c_int, [_vp, _ip, _ip, _ip, _ip, _ip, _ip64]),
    "isvd_engine_has_reference": (C.c_int, [_vp, _ip, _ip, _ip]),
    "isvd_engine_get_factors": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp]),
    "isvd_engine_get_tracked": (C.c_int, [_vp, C.c_int, _dp]),
    "isvd_engine_get_reference": (C.c_int, [_vp, C.c_int, _dp]),
    "isvd_engine_get_scalars": (C.c_int, [_vp, _dp, _dp, _dp]),
    "isvd_engine_set_factors": (C.c_int, [_vp, C.c_int, C.c_int, _dp, _dp, _dp]),
    "isvd_engine_put_reference": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _dp]),
    "isvd_engine_device_views": (C.c_int, [_vp, C.POINTER(_vp), _ip64, _ip, C.POINTER(_vp), _ip64,
                                           _ip, C.POINTER(_vp), _ip, C.POINTER(_vp), _ip64, _ip]),
    "isvd_engine_canonicalize": (C.c_int, [_vp]),
    "isvd_engine_stream": (_vp, [_vp]),
    "isvd_ortho_defect": (C.c_int, [C.c_int, C.c_int, C.c_int, _dp, _dp]),
    "isvd_principal_angle": (C.c_int, [C.c_int, C.c_int, _dp, _dp, _dp]),
    "isvd_engine_streams": (C.c_int, [_vp, C.POINTER(_vp), C.c_int]),
    "isvd_engine_synchronize": (C.c_int, [_vp]),
    "isvd_engine_set_timing": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_set_append_solver": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_set_lazy": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_risk": (C.c_int, [_vp, C.c_int, _dp, C.c_int, _dp, _dp, _dp]),
    "isvd_low_rank_cov": (C.c_int, [C.c_int, C.c_int, _dp, _dp, C.c_int, _dp]),
    "isvd_engine_scalars_async": (C.c_int, [_vp, _vp, C.c_int]),
    "isvd_engine_scalars_wait": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_set_shard": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int,
                                        C.c_void_p, C.c_void_p]),
    "isvd_engine_shard_info": (C.c_int, [_vp, _ip64, _ip, _ip]),
    "isvd_engine_set_lazy_window": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_lazy_window": (C.c_int, [_vp]),
    "isvd_engine_set_vdefer": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_set_groups": (C.c_int, [_vp, C.c_int]),
    "isvd_engine_set_reortho_threshold": (C.c_int, [_vp, C.c_double]),
    "isvd_engine_flush": (C.c_int, [_vp]),
    "isvd_engine_snapshot": (C.c_int, [_vp]),
    "isvd_engine_restore": (C.c_int, [_vp]),
    "isvd_engine_phase_times": (C.c_int, [_vp, _dp, _ip64]),
    "isvd_engine_frob_error": (C.c_int, [_vp, _dp]),
    "isvd_engine_ortho_defect": (C.c_int, [_vp, _dp, _dp]),
    "isvd_engine_angle": (C.c_int, [_vp, C.c_int, _vp, C.c_int, C.c_int, _dp]),
    "isvd_dense_svd": (C.c_int, [C.c_int, C.c_int, C.c_int, _dp, C.c_int, _dp, _dp, _dp]),
    "isvd_gram": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int, _vp, C.c_int, _vp, _vp]),
    "isvd_gemm_tall": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int, _vp, C.c_int, _vp, C.c_int, _vp]),
    "isvd_engine_oracle": (C.c_int, [_vp, C.c_int, _dp, _dp]),
}

_lib = None


def load() -> C.CDLL:
    """Load libisvd.so (raising loudly if it is absent)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2605_24514_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class IsvdError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map a C status to the reference's exception types."""
    if rc == ISVD_OK:
        return
    msg = load().isvd_last_error().decode(errors="replace")
    if rc == ISVD_EINVAL:
        raise ValueError(msg)
    raise IsvdError(f"libisvd error {rc}: {msg}")


def dptr(a: np.ndarray):
    """double* of a C-contiguous float64 numpy array."""
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def vptr(a) -> int:
    """void* of a numpy array or a torch tensor (device or host)."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


# int (*)(void* ctx, double* buf, int64_t count, void* stream)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


def launch_count() -> int:
    return int(load().isvd_launch_count())
