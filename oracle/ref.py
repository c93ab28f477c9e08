"""oracle/ref.py -- TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/_ref/libcoserve_ref.so: the reference's own headers
(tiny_model.hpp, rng.hpp, matrix.hpp) compiled unmodified by oracle/Makefile.
Used to pin oracle/coserve_oracle.py and as bench.py's CPU baseline
(cpu_baseline.kind == "reference").  Absent on machines where neither the
reference tree nor a prebuilt _ref/ exists: `available()` says so.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "_ref", "libcoserve_ref.so")
_LIB = None


def _cpu_flags() -> set:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def march() -> str:
    """Highest x86-64 micro-architecture level of the prebuilt reference this host can run."""
    fl = _cpu_flags()
    if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= fl and \
            os.path.exists(_PATH.replace(".so", "_v4.so")):
        return "x86-64-v4"
    if {"avx2", "fma", "bmi2"} <= fl and os.path.exists(_PATH.replace(".so", "_v3.so")):
        return "x86-64-v3"
    return "x86-64-v2"


def path() -> str:
    lvl = march()
    return {"x86-64-v4": _PATH.replace(".so", "_v4.so"),
            "x86-64-v3": _PATH.replace(".so", "_v3.so")}.get(lvl, _PATH)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def available() -> bool:
    return os.path.exists(_PATH)


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise FileNotFoundError(f"{_PATH} not built (reference tree absent?)")
        L = ctypes.CDLL(path())
        vp, i, l, u64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_long, ctypes.c_uint64, ctypes.c_double
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_model_init.restype = vp
        L.ref_model_init.argtypes = [i, l, i, l, l, i, u64]
        L.ref_model_free.argtypes = [vp]
        L.ref_model_get.restype = l
        L.ref_model_get.argtypes = [vp, ctypes.c_char_p, i, vp]
        L.ref_model_set.restype = l
        L.ref_model_set.argtypes = [vp, ctypes.c_char_p, i, vp]
        L.ref_forward_backward.restype = i
        L.ref_forward_backward.argtypes = [vp, vp, l] + [vp] * 8
        L.ref_time_forward_backward.restype = d
        L.ref_time_forward_backward.argtypes = [vp, vp, l, i]
        L.ref_rng_uniform_int.argtypes = [u64, l, l, l, vp]
        L.ref_rng_normal.argtypes = [u64, l, vp]
        L.ref_rng_mixed.argtypes = [u64, l, vp]
        _LIB = L
    return _LIB


class RefTinyModel:
    """TinyModel (tiny_model.hpp:38-68) living inside the reference build."""

    def __init__(self, depth=2, hidden=16, heads=1, ffn_mult=4, vocab=64, rank=2, seed=1):
        self.depth, self.hidden, self.heads = depth, hidden, heads
        self.ffn, self.vocab, self.rank = hidden * ffn_mult, vocab, rank
        self._h = lib().ref_model_init(depth, hidden, heads, ffn_mult, vocab, rank, seed)
        if not self._h:
            raise ValueError(lib().ref_last_error().decode())

    def __del__(self):
        try:
            lib().ref_model_free(self._h)
        except Exception:
            pass

    def _shape(self, name):
        h, f, r, V = self.hidden, self.ffn, self.rank, self.vocab
        return {"embed": (V, h), "unembed": (h, V), "wq": (h, h), "wk": (h, h), "wv": (h, h),
                "wo": (h, h), "w_up": (h, f), "w_down": (f, h), "lora_a": (f, r),
                "lora_b": (r, h)}[name]

    def get(self, name: str, layer: int = 0) -> np.ndarray:
        out = np.zeros(self._shape(name))
        n = lib().ref_model_get(self._h, name.encode(), layer, out.ctypes.data)
        assert n == out.size
        return out

    def set(self, name: str, layer: int, value: np.ndarray):
        v = np.ascontiguousarray(value, dtype=np.float64)
        n = lib().ref_model_set(self._h, name.encode(), layer, v.ctypes.data)
        assert n == v.size

    def weights(self) -> Dict:
        W = {"embed": self.get("embed"), "unembed": self.get("unembed"), "layers": []}
        for l in range(self.depth):
            W["layers"].append({k: self.get(k, l) for k in
                                ("wq", "wk", "wv", "wo", "w_up", "w_down", "lora_a", "lora_b")})
        return W

    def forward_backward(self, tokens, backward=True) -> Dict:
        toks = np.ascontiguousarray(tokens, dtype=np.int32)
        L = len(toks)
        h, f, r, V, N = self.hidden, self.ffn, self.rank, self.vocab, self.depth
        loss = np.zeros(1)
        logits = np.zeros((L, V))
        fh = np.zeros((L, h))
        ga = np.zeros((N, f, r)) if backward else None
        gb = np.zeros((N, r, h)) if backward else None
        dk = np.zeros((N, L, h)) if backward else None
        dv = np.zeros((N, L, h)) if backward else None
        dx = np.zeros((N, L, h)) if backward else None
        p = lambda a: None if a is None else a.ctypes.data
        rc = lib().ref_forward_backward(self._h, toks.ctypes.data, L, p(loss), p(logits), p(fh),
                                        p(ga), p(gb), p(dk), p(dv), p(dx))
        if rc != 0:
            raise ValueError(lib().ref_last_error().decode())
        return {"loss": float(loss[0]), "logits": logits, "final_hidden": fh,
                "grad_a": ga, "grad_b": gb, "dk": dk, "dv": dv, "dx": dx}

    def time_forward_backward(self, tokens, iters: int) -> float:
        toks = np.ascontiguousarray(tokens, dtype=np.int32)
        return lib().ref_time_forward_backward(self._h, toks.ctypes.data, len(toks), iters)


def rng_uniform_int(seed: int, n: int, lo: int, hi: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.int64)
    lib().ref_rng_uniform_int(seed, n, lo, hi, out.ctypes.data)
    return out


def rng_normal(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    lib().ref_rng_normal(seed, n, out.ctypes.data)
    return out


def rng_mixed(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    lib().ref_rng_mixed(seed, n, out.ctypes.data)
    return out
