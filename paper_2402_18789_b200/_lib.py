"""ctypes binding of libcoserve_cuda.so (the product's C ABI, include/coserve_cuda.h).

Fails loudly if the in-tree library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# CS_TRACE_LIB=1: the -DCS_TRACE build (in-kernel event timelines; scripts/trace_bwd.py only)
# CS_LIB_PATH: an experiment variant built by scripts/build_variant.py
LIB_PATH = os.environ.get("CS_LIB_PATH") or os.path.join(
    _PKG, "libcoserve_cuda_trace.so" if os.environ.get("CS_TRACE_LIB") == "1" else "libcoserve_cuda.so")
_LIB = None


class CoserveError(RuntimeError):
    pass


class CacheDesync(CoserveError):
    pass


class OrderingViolation(CoserveError):
    pass


CS_OK = 0
CS_ERR_INVALID_ARGUMENT = -1
CS_ERR_RUNTIME = -2
CS_ERR_CUDA = -3
CS_ERR_CACHE_DESYNC = -4
CS_ERR_ORDERING = -5
CS_ERR_OOM = -6
CS_ERR_NCCL = -7


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2402_18789_b200.build` "
                "(no CPU fallback exists for the co-serving path)")
        _LIB = ctypes.CDLL(LIB_PATH)
        _declare(_LIB)
    return _LIB


def _declare(L):
    vp, i32, i64, f32, f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                              ctypes.c_double)
    L.cs_last_error.restype = ctypes.c_char_p
    L.cs_version.restype = ctypes.c_int
    L.cs_gemm_bf16.restype = ctypes.c_int
    L.cs_gemm_bf16.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, ctypes.c_int, vp,
                               ctypes.c_int, ctypes.c_int, vp]
    L.cs_gemm_bf16_mn.restype = ctypes.c_int
    L.cs_gemm_bf16_mn.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, vp]


def check(rc: int, what: str = ""):
    if rc == CS_OK:
        return
    msg = lib().cs_last_error().decode()
    if rc == CS_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == CS_ERR_CACHE_DESYNC:
        raise CacheDesync(msg)
    if rc == CS_ERR_ORDERING:
        raise OrderingViolation(msg)
    raise CoserveError(f"{what} failed ({rc}): {msg}")
