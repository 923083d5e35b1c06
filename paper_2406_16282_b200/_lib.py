"""ctypes loader for liblmbp.so (the C ABI declared in include/lmbp.h).

There is no fallback: if the library is missing or cannot be loaded, importing
anything that needs it raises.  Build it with
``python -m paper_2406_16282_b200.build`` (``__graft_entry__.build()`` does).
"""
from __future__ import annotations

import ctypes
import os

from .build import LIB

_p, _i64, _i32, _f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
_f64, _u64 = ctypes.c_double, ctypes.c_uint64

# name -> (restype, argtypes); mirrors include/lmbp.h
SIGNATURES = {
    "lmbp_codes_bytes": (ctypes.c_size_t, [_i64]),
    "lmbp_status_string": (ctypes.c_char_p, [_i32]),
    "lmbp_version": (ctypes.c_char_p, []),
    "lmbp_step_table": (_i32, [_i32, _p, _p]),
    "regelu2_fwd": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p]),
    "regelu2_bwd": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p]),
    "resilu2_fwd": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p]),
    "resilu2_bwd": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p]),
    "msln_fwd": (_i32, [_p, _p, _p, _i64, _i64, _f32, _i32, _p]),
    "msln_bwd": (_i32, [_p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "msrms_fwd": (_i32, [_p, _p, _p, _i64, _i64, _f32, _i32, _p]),
    "msrms_bwd": (_i32, [_p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "msln_fwd_mixed": (_i32, [_p, _p, _p, _i64, _i64, _f32, _i32, _p]),
    "msln_bwd_mixed": (_i32, [_p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "msrms_fwd_mixed": (_i32, [_p, _p, _p, _i64, _i64, _f32, _i32, _p]),
    "msrms_bwd_mixed": (_i32, [_p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "reswiglu2_fwd": (_i32, [_p, _p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "lmbp_codes_bytes_k": (ctypes.c_size_t, [_i64, _i32]),
    "stepact_fwd": (_i32, [_i32, _i32, _p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "stepact_bwd": (_i32, [_i32, _p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "reswiglu2_bwd": (_i32, [_p, _p, _p, _p, _p, _p, _i64, _i64, _i32, _p]),
    "lmbp_fit_bounds": (_i32, [_i32, _f64, _p, _p]),
    "lmbp_fit_objective": (_i32, [_i32, _i32, _i32, _f64, _p, _p, _i64, _p]),
    "lmbp_fit_refine": (_i32, [_i32, _i32, _i32, _f64, _p, _i64, _i64, _p, _p, _p, _p]),
    "lmbp_fit_anneal_vp": (_i32, [_i32, _i32, _i32, _f64, _p, _i64, _i64, _u64, _f64, _f64, _f64, _f64, _p, _p,
                                  _p, _p]),
    "lmbp_fit_anneal": (_i32, [_i32, _i32, _i32, _f64, _p, _i64, _i64, _u64, _f64, _f64, _f64, _f64, _p, _p, _p,
                               _p]),
}

(LMBP_OK, LMBP_ERR_NULLPTR, LMBP_ERR_SHAPE, LMBP_ERR_DTYPE, LMBP_ERR_EPS, LMBP_ERR_CUDA, LMBP_ERR_KIND,
 LMBP_ERR_TABLE, LMBP_ERR_ARG) = range(9)
LMBP_FIT_H, LMBP_FIT_DH = 0, 1
LMBP_F32, LMBP_BF16, LMBP_F16 = 0, 1, 2
LMBP_GELU, LMBP_SILU = 0, 1

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded liblmbp.so.  Raises if it is absent -- never falls back."""
    global _lib
    if _lib is None:
        # LMBP_LIBRARY: a tuning build of the same sources with extra -D
        # defines (build.build_variant, built without the fitter) for A/B runs
        # of bench.py; the product library otherwise.
        path = os.environ.get("LMBP_LIBRARY") or LIB
        if not os.path.exists(path):
            raise ImportError(f"liblmbp.so not found at {path}; run `python -m paper_2406_16282_b200.build` "
                              "(no CPU fallback exists)")
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name, None)
            if f is None and path != LIB and name.startswith("lmbp_fit"):
                continue
            if f is None:
                raise ImportError(f"{path} does not export {name}")
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().lmbp_status_string(int(status)).decode()


class LmbpError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        super().__init__(f"{fn}: {status_string(status)}")


def check(fn: str, status: int) -> None:
    if status != LMBP_OK:
        raise LmbpError(fn, status)
