"""oracle/coserve_oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

CPU f64 restatement of the reference's hot-path arithmetic, in numpy:

  * Rng                      rng.hpp:15-64           (via oracle/_build/liborc_rng.so, a C restatement)
  * init_tiny                tiny_model.hpp:44-67    (draw order + scales; LoRA B non-zero)
  * forward_full             tiny_model.hpp:181-221  (embed -> N x [QKV, causal MHA, O, resid,
                                                      up, ReLU, down + LoRA(A,B), resid] -> unembed -> mean CE)
  * backward_full            tiny_model.hpp:248-327  (LoRA grads, dK/dV/dX per layer; frozen dW never formed)
  * loss_head_grad           tiny_model.hpp:223-246
  * max_rel_err / rel_err    matrix.hpp:127-139
  * forward_window / backward_window / generative_loss / QkvCache / KvGradAccumulator
                             SPEC.md:248-309 (Alg. 2; Slice read as [l_j-s_j, l_j))

and the north_star-only LLaMA/Qwen generalisation the reference cannot express
(SURVEY.md §8 a21): RMSNorm, rotate-half RoPE, SwiGLU, GQA, QKV bias.  With
arch.norm == 'none', arch.act == 'relu', no RoPE, Hkv == Hq and no bias the
general code path reduces to the reference's exact op sequence, which the tests
pin against the reference itself (oracle/_ref) and SURVEY.md Appendix A.

bf16 rounding-point emulation (emu=True on forward_full / backward_full / forward_window /
backward_window): the same op sequence with every value rounded to bf16 where the GPU path
stores or feeds bf16 -- frozen weights and the LoRA A/B copies as GEMM operands, normed
activations, Q/K/V (after RoPE), P and dS inside attention, attention output, gate/up and the
MLP activation, bf16(u) in the K-concatenated down GEMM, dlogits, dY / dU / dm / dgu / dr1 / dO /
dqkv in the backward -- and fp32-like accumulation everywhere else (f64 here).  It isolates
the GPU's kernel arithmetic from the bf16 storage floor: tests gate the GPU against it at
rel <= 1e-2 (north_star) and report the f64 comparison as the floor.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_RNG_LIB = None


_BFW_CACHE: Dict[int, tuple] = {}


def bfw(x):
    """Round to bf16 (round-to-nearest-even on the fp32 bit pattern, as __float2bfloat16_rn)
    and return float64: a weight operand of the emu oracle.  Large weight arrays are rounded
    once and memoised (by identity; the cache holds the array so the id stays unique) -- only
    persistent weight arrays may go through here, never temporaries, and they must not be
    mutated in place while cached (clear_weight_cache)."""
    if isinstance(x, np.ndarray) and x.size >= (1 << 20):
        hit = _BFW_CACHE.get(id(x))
        if hit is not None and hit[0] is x:
            return hit[1]
        r = _bfw(x)
        _BFW_CACHE[id(x)] = (x, r)
        return r
    return _bfw(x)


def clear_weight_cache():
    _BFW_CACHE.clear()


def _bfw(x):
    a = np.array(x, dtype=np.float32, copy=True, order="C")
    u = a.view(np.uint32)
    # round-to-nearest-even on the upper 16 bits; no uint32 overflow for finite values
    lsb = (u >> 16) & 1
    u += 0x7FFF
    u += lsb
    u &= 0xFFFF0000
    return a.astype(np.float64)


_NOISE = None  # (rng, relative amplitude): emu_sensitivity's fp32-level perturbation


def bf16(x):
    """bf16 at an activation rounding point of the emu oracle (the GPU's bf16 stores)."""
    if _NOISE is not None:
        rng, amp = _NOISE
        x = np.asarray(x, dtype=np.float64)
        x = x * (1.0 + amp * rng.standard_normal(x.shape))
    return _bfw(x)


def emu_sensitivity(arch, W, tokens, amp: float = 3e-7, trials: int = 3, seed: int = 0,
                    clean=None):
    """How far two bf16 evaluations of the same model drift apart when their pre-rounding
    activations differ only at fp32 level (relative noise `amp` ~ a few fp32 ulps, i.e. fp32
    vs f64 accumulation): max over trials of the scale-normalised deviation of every backward
    quantity from the noise-free emu run.  Where this exceeds 1e-2 (the reference arch's ReLU:
    a unit with up ~ 0 flips its mask, tiny_model.hpp:285-286, and passes or blocks a whole
    gradient row) no bf16 implementation can be held to 1e-2 of another; tests use it as the
    floor for those quantities."""
    global _NOISE
    if clean is None:  # the noise-free emu backward of the same case (or pass it in)
        clean = backward_full(arch, W, forward_full(arch, W, tokens, emu=True))
    be = clean
    out = {}
    try:
        _NOISE = (np.random.default_rng(seed), amp)
        for _ in range(trials):
            t2 = forward_full(arch, W, tokens, emu=True)
            b2 = backward_full(arch, W, t2)
            q = {}
            for l in range(arch.n_layers):
                q[f"dA{l}"] = scaled_err(b2["grads"]["a"][l], be["grads"]["a"][l])
                q[f"dB{l}"] = scaled_err(b2["grads"]["b"][l], be["grads"]["b"][l])
                for k in ("dk", "dv", "dx"):
                    q[f"d{k[1].upper()}{l}"] = scaled_err(b2["layers"][l][k], be["layers"][l][k])
            for k, v in q.items():
                out[k] = max(out.get(k, 0.0), v)
    finally:
        _NOISE = None
    return out


def _rng_lib():
    global _RNG_LIB
    if _RNG_LIB is None:
        path = os.path.join(_HERE, "_build", "liborc_rng.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", _HERE, "_build/liborc_rng.so"])
        lib = ctypes.CDLL(path)
        vp, u64, i64, d = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
        lib.orc_rng_new.restype = vp
        lib.orc_rng_new.argtypes = [u64]
        lib.orc_rng_free.argtypes = [vp]
        lib.orc_rng_bits.restype = u64
        lib.orc_rng_bits.argtypes = [vp]
        lib.orc_rng_uniform.restype = d
        lib.orc_rng_uniform.argtypes = [vp]
        lib.orc_rng_uniform_int.argtypes = [vp, i64, i64, i64, vp]
        lib.orc_rng_normal.restype = d
        lib.orc_rng_normal.argtypes = [vp]
        lib.orc_rng_lognormal.restype = d
        lib.orc_rng_lognormal.argtypes = [vp, d, d]
        lib.orc_rng_exponential.restype = d
        lib.orc_rng_exponential.argtypes = [vp, d]
        lib.orc_rng_randn.argtypes = [vp, i64, i64, d, vp]
        _RNG_LIB = lib
    return _RNG_LIB


class Rng:
    """rng.hpp:15-64 (mt19937_64 + hand-rolled distributions)."""

    def __init__(self, seed: int):
        self._lib = _rng_lib()
        self._h = self._lib.orc_rng_new(ctypes.c_uint64(seed))

    def __del__(self):
        try:
            self._lib.orc_rng_free(self._h)
        except Exception:
            pass

    def bits(self) -> int:
        return int(self._lib.orc_rng_bits(self._h))

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lo + (hi - lo) * self._lib.orc_rng_uniform(self._h)

    def uniform_int(self, lo: int, hi: int, n: Optional[int] = None):
        k = 1 if n is None else n
        out = np.zeros(k, dtype=np.int64)
        self._lib.orc_rng_uniform_int(self._h, lo, hi, k, out.ctypes.data)
        return int(out[0]) if n is None else out

    def normal(self) -> float:
        return self._lib.orc_rng_normal(self._h)

    def lognormal(self, mu: float, sigma: float) -> float:
        return self._lib.orc_rng_lognormal(self._h, mu, sigma)

    def exponential(self, rate: float) -> float:
        return self._lib.orc_rng_exponential(self._h, rate)

    def randn(self, rows: int, cols: int, scale: float) -> np.ndarray:
        out = np.zeros((rows, cols), dtype=np.float64)
        self._lib.orc_rng_randn(self._h, rows, cols, scale, out.ctypes.data)
        return out


# ---------------------------------------------------------------------------
# Architecture + weights
# ---------------------------------------------------------------------------

@dataclass
class Arch:
    """Generalised TinyModelConfig (tiny_model.hpp:17-28) with the LLaMA/Qwen knobs
    the reference cannot express (SURVEY.md §5 'Config / flags')."""
    n_layers: int = 2
    hidden: int = 16
    n_heads: int = 1
    n_kv_heads: int = 1
    head_dim: int = 16
    ffn: int = 64
    vocab: int = 64
    lora_rank: int = 2
    norm: str = "none"      # 'none' (reference) | 'rms'
    act: str = "relu"       # 'relu' (reference, up only) | 'swiglu' (gate || up)
    rope: bool = False
    qkv_bias: bool = False
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5

    @property
    def q_dim(self):
        return self.n_heads * self.head_dim

    @property
    def kv_dim(self):
        return self.n_kv_heads * self.head_dim

    @staticmethod
    def reference(depth=2, hidden=16, heads=1, ffn_mult=4, vocab=64, rank=2) -> "Arch":
        return Arch(n_layers=depth, hidden=hidden, n_heads=heads, n_kv_heads=heads,
                    head_dim=hidden // heads, ffn=hidden * ffn_mult, vocab=vocab,
                    lora_rank=rank)

    def is_reference(self) -> bool:
        return (self.norm == "none" and self.act == "relu" and not self.rope
                and not self.qkv_bias and self.n_kv_heads == self.n_heads
                and self.q_dim == self.hidden)


LAYER_KEYS = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down", "lora_a", "lora_b",
              "bq", "bk", "bv", "g1", "g2")


def init_tiny(arch: Arch, seed: int = 1) -> Dict:
    """TinyModel::init, tiny_model.hpp:44-67: one Rng(seed) stream, row-major randn in
    the order embed, unembed, then per layer wq, wk, wv, wo, w_up, w_down, lora_a, lora_b."""
    if arch.hidden % arch.n_heads != 0:
        raise ValueError("tiny model: heads must divide hidden")  # :45-46
    if arch.lora_rank < 1:
        raise ValueError("tiny model: rank must be >= 1")  # :47
    assert arch.is_reference()
    h, f, r, V = arch.hidden, arch.ffn, arch.lora_rank, arch.vocab
    rng = Rng(seed)
    ws = 1.0 / math.sqrt(float(h))
    W = {"embed": rng.randn(V, h, ws), "unembed": rng.randn(h, V, ws), "layers": []}
    for _ in range(arch.n_layers):
        L = {}
        L["wq"] = rng.randn(h, h, ws)
        L["wk"] = rng.randn(h, h, ws)
        L["wv"] = rng.randn(h, h, ws)
        L["wo"] = rng.randn(h, h, ws)
        L["w_up"] = rng.randn(h, f, ws)
        L["w_down"] = rng.randn(f, h, 1.0 / math.sqrt(float(f)))
        L["lora_a"] = rng.randn(f, r, 0.2 / math.sqrt(float(f)))
        L["lora_b"] = rng.randn(r, h, 0.2)
        W["layers"].append(L)
    return W


def init_general(arch: Arch, seed: int = 1) -> Dict:
    """Deterministic init for LLaMA-style test archs, same scale scheme as the reference
    (N(0,1/h); w_down N(0,1/f); A N(0,(0.2/sqrt f)^2); B N(0,0.2^2)); norm gains near 1."""
    rng = np.random.default_rng(seed)
    h, f, r, V = arch.hidden, arch.ffn, arch.lora_rank, arch.vocab
    ws = 1.0 / math.sqrt(h)
    W = {"embed": rng.standard_normal((V, h)) * ws,
         "unembed": rng.standard_normal((h, V)) * ws, "layers": []}
    if arch.norm == "rms":
        W["gf"] = 1.0 + 0.1 * rng.standard_normal(h)
    for _ in range(arch.n_layers):
        L = {"wq": rng.standard_normal((h, arch.q_dim)) * ws,
             "wk": rng.standard_normal((h, arch.kv_dim)) * ws,
             "wv": rng.standard_normal((h, arch.kv_dim)) * ws,
             "wo": rng.standard_normal((arch.q_dim, h)) * (1.0 / math.sqrt(arch.q_dim)),
             "w_up": rng.standard_normal((h, f)) * ws,
             "w_down": rng.standard_normal((f, h)) * (1.0 / math.sqrt(f)),
             "lora_a": rng.standard_normal((f, r)) * (0.2 / math.sqrt(f)),
             "lora_b": rng.standard_normal((r, h)) * 0.2}
        if arch.act == "swiglu":
            L["w_gate"] = rng.standard_normal((h, f)) * ws
        if arch.qkv_bias:
            L["bq"] = 0.1 * rng.standard_normal(arch.q_dim)
            L["bk"] = 0.1 * rng.standard_normal(arch.kv_dim)
            L["bv"] = 0.1 * rng.standard_normal(arch.kv_dim)
        if arch.norm == "rms":
            L["g1"] = 1.0 + 0.1 * rng.standard_normal(h)
            L["g2"] = 1.0 + 0.1 * rng.standard_normal(h)
        W["layers"].append(L)
    return W


# ---------------------------------------------------------------------------
# Elementwise pieces (LLaMA generalisation; identity for the reference arch)
# ---------------------------------------------------------------------------

def rms_fwd(x, g, eps):
    rstd = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * rstd * g, rstd


def rms_bwd(x, g, rstd, dy):
    n = x.shape[-1]
    xhat = x * rstd
    dxhat = dy * g
    return rstd * (dxhat - xhat * np.sum(dxhat * xhat, axis=-1, keepdims=True) / n)


def rope_tables(positions, d, theta):
    half = d // 2
    inv = theta ** (-(np.arange(half, dtype=np.float64) * 2.0) / d)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope_apply(x, positions, n_heads, d, theta, inverse=False):
    """rotate-half RoPE on [s, n_heads*d]; inverse=True applies the transpose (backward)."""
    if x.shape[0] == 0:
        return x.copy()
    c, s = rope_tables(positions, d, theta)
    if inverse:
        s = -s
    xr = x.reshape(x.shape[0], n_heads, d)
    x1, x2 = xr[..., : d // 2], xr[..., d // 2:]
    c, s = c[:, None, :], s[:, None, :]
    out = np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)
    return out.reshape(x.shape)


def silu(x):
    return x / (1.0 + np.exp(-x))


def dsilu(x):
    sg = 1.0 / (1.0 + np.exp(-x))
    return sg * (1.0 + x * (1.0 - sg))


# ---------------------------------------------------------------------------
# Caches
# ---------------------------------------------------------------------------

@dataclass
class LayerSaved:
    """Per-layer per-position activations (the oracle keeps everything; the GPU path
    keeps only what survives graph pruning)."""
    x_in: np.ndarray
    q: np.ndarray   # roped
    k: np.ndarray   # roped
    v: np.ndarray
    r1: np.ndarray
    pre: np.ndarray  # relu: up ; swiglu: gate
    up: np.ndarray   # swiglu: up ; relu: unused
    m: np.ndarray    # MLP activation (relu_out / silu(g)*u)
    lu: np.ndarray   # LoRA u = m @ A
    rstd1: np.ndarray
    rstd2: np.ndarray
    o: Optional[np.ndarray] = None  # attention output (emu: the bf16 O the GPU saves for Delta)


class QkvCache:
    """per-layer Q, K, V of all processed positions, growing monotonically."""

    def __init__(self, arch: Arch, max_len: int):
        self.arch = arch
        self.length = 0
        n = arch.n_layers
        z = lambda c: [np.zeros((max_len, c)) for _ in range(n)]
        self.saved = [LayerSaved(x_in=np.zeros((max_len, arch.hidden)),
                                 q=np.zeros((max_len, arch.q_dim)),
                                 k=np.zeros((max_len, arch.kv_dim)),
                                 v=np.zeros((max_len, arch.kv_dim)),
                                 r1=np.zeros((max_len, arch.hidden)),
                                 pre=np.zeros((max_len, arch.ffn)),
                                 up=np.zeros((max_len, arch.ffn)),
                                 m=np.zeros((max_len, arch.ffn)),
                                 lu=np.zeros((max_len, arch.lora_rank)),
                                 rstd1=np.zeros((max_len, 1)), rstd2=np.zeros((max_len, 1)),
                                 o=np.zeros((max_len, arch.q_dim)))
                      for _ in range(n)]
        del z


class KvGradAccumulator:
    """SPEC.md:253-257 (ΔKVAccum): per-layer dK, dV [L, kv_dim] (in roped-K space)."""

    def __init__(self, arch: Arch, L: int):
        self.dk = [np.zeros((L, arch.kv_dim)) for _ in range(arch.n_layers)]
        self.dv = [np.zeros((L, arch.kv_dim)) for _ in range(arch.n_layers)]


class CacheDesync(RuntimeError):
    pass


class OrderingViolation(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# Forward over a window of rows (attention_rows generalised; tiny_model.hpp:118-151)
# ---------------------------------------------------------------------------

def _attention_rows(arch: Arch, q, K, V, row_begin, emu: bool = False):
    """q: [s, Hq*d] rows at positions row_begin.., K/V: [row_begin+s, Hkv*d].
    Returns out [s, Hq*d] and lse [s, Hq] (the GPU saves LSE instead of probs).
    emu: unnormalised P rounded to bf16 for the PV product, fp32-style row sum, bf16 output."""
    s = q.shape[0]
    d, Hq, Hkv = arch.head_dim, arch.n_heads, arch.n_kv_heads
    grp = Hq // Hkv
    scale = 1.0 / math.sqrt(float(d))
    out = np.zeros((s, Hq * d))
    lse = np.zeros((s, Hq))
    e = row_begin + s
    mask = np.arange(e)[None, :] <= (row_begin + np.arange(s))[:, None]  # [s, e]
    for hq in range(Hq):
        hk = hq // grp
        qh = q[:, hq * d:(hq + 1) * d]
        kh = K[:e, hk * d:(hk + 1) * d]
        vh = V[:e, hk * d:(hk + 1) * d]
        sc = (qh @ kh.T) * scale
        sc = np.where(mask, sc, -np.inf)
        mx = sc.max(axis=1, keepdims=True)
        p = np.exp(sc - mx)
        den = p.sum(axis=1, keepdims=True)
        if emu:
            out[:, hq * d:(hq + 1) * d] = (bf16(p) @ vh) / den
        else:
            p /= den
            out[:, hq * d:(hq + 1) * d] = p @ vh
        lse[:, hq] = (mx + np.log(den))[:, 0]
    return (bf16(out) if emu else out), lse


def _layer_forward(arch: Arch, w: Dict, x, pos0: int, sv: LayerSaved, lora: bool = True,
                   ar=None, emu: bool = False):
    """ar: tensor-parallel all-reduce of the row-parallel partial sums (oracle/tp_oracle.py);
    None = one rank, reference op order.  emu: bf16 rounding points of the GPU path."""
    if emu:
        return _layer_forward_emu(arch, w, x, pos0, sv, lora)
    s = x.shape[0]
    rows = slice(pos0, pos0 + s)
    positions = np.arange(pos0, pos0 + s)
    sv.x_in[rows] = x
    if arch.norm == "rms":
        h1, r = rms_fwd(x, w["g1"], arch.rms_eps)
        sv.rstd1[rows] = r
    else:
        h1 = x
    q = h1 @ w["wq"]
    k = h1 @ w["wk"]
    v = h1 @ w["wv"]
    if arch.qkv_bias:
        q = q + w["bq"]
        k = k + w["bk"]
        v = v + w["bv"]
    if arch.rope:
        q = rope_apply(q, positions, arch.n_heads, arch.head_dim, arch.rope_theta)
        k = rope_apply(k, positions, arch.n_kv_heads, arch.head_dim, arch.rope_theta)
    sv.q[rows], sv.k[rows], sv.v[rows] = q, k, v
    attn, _ = _attention_rows(arch, q, sv.k, sv.v, pos0)
    r1 = x + (attn @ w["wo"] if ar is None else ar(attn @ w["wo"]))  # tiny_model.hpp:201-202
    sv.r1[rows] = r1
    if arch.norm == "rms":
        h2, r = rms_fwd(r1, w["g2"], arch.rms_eps)
        sv.rstd2[rows] = r
    else:
        h2 = r1
    if arch.act == "relu":
        up = h2 @ w["w_up"]                                  # :203
        m = np.where(up > 0.0, up, 0.0)                      # :204-205
        sv.pre[rows] = up
    else:
        g = h2 @ w["w_gate"]
        u = h2 @ w["w_up"]
        m = silu(g) * u
        sv.pre[rows], sv.up[rows] = g, u
    sv.m[rows] = m
    if ar is not None:  # TP: u = m_r A_r partial, its up-projection folded into the down sum
        delta = m @ w["w_down"]
        if lora:
            lu = m @ w["lora_a"]
            sv.lu[rows] = lu
            delta = delta + lu @ w["lora_b"]
        return r1 + ar(delta)
    y = r1 + m @ w["w_down"]                                 # :209-210
    if lora:  # inference rows of a base-model request skip the adapter (segmented LoRA)
        lu = m @ w["lora_a"]                                 # :207
        sv.lu[rows] = lu
        y = y + lu @ w["lora_b"]                             # :208,211
    return y


def _layer_forward_emu(arch: Arch, w: Dict, x, pos0: int, sv: LayerSaved, lora: bool):
    """_layer_forward with the GPU path's bf16 storage points (engine.cu:forward): residual x
    fp32, GEMM operands bf16, fp32 accumulation; QKV (+bias) rounded in the GEMM epilogue,
    RoPE applied to the bf16 values and rounded again (rope_append_kernel)."""
    s = x.shape[0]
    rows = slice(pos0, pos0 + s)
    positions = np.arange(pos0, pos0 + s)
    sv.x_in[rows] = x
    if arch.norm == "rms":
        h1, r = rms_fwd(x, w["g1"], arch.rms_eps)
        sv.rstd1[rows] = r
    else:
        h1 = x
    h1 = bf16(h1)
    q, k, v = h1 @ bfw(w["wq"]), h1 @ bfw(w["wk"]), h1 @ bfw(w["wv"])
    if arch.qkv_bias:
        q, k, v = q + w["bq"], k + w["bk"], v + w["bv"]
    q, k, v = bf16(q), bf16(k), bf16(v)
    if arch.rope:
        q = bf16(rope_apply(q, positions, arch.n_heads, arch.head_dim, arch.rope_theta))
        k = bf16(rope_apply(k, positions, arch.n_kv_heads, arch.head_dim, arch.rope_theta))
    sv.q[rows], sv.k[rows], sv.v[rows] = q, k, v
    attn, _ = _attention_rows(arch, q, sv.k, sv.v, pos0, emu=True)
    sv.o[rows] = attn
    r1 = x + attn @ bfw(w["wo"])
    sv.r1[rows] = r1
    if arch.norm == "rms":
        h2, r = rms_fwd(r1, w["g2"], arch.rms_eps)
        sv.rstd2[rows] = r
    else:
        h2 = r1
    h2 = bf16(h2)
    if arch.act == "relu":
        up = bf16(h2 @ bfw(w["w_up"]))
        m = np.where(up > 0.0, up, 0.0)
        sv.pre[rows] = up
    else:
        g = bf16(h2 @ bfw(w["w_gate"]))
        u = bf16(h2 @ bfw(w["w_up"]))
        m = bf16(silu(g) * u)
        sv.pre[rows], sv.up[rows] = g, u
    sv.m[rows] = m
    y = r1 + m @ bfw(w["w_down"])
    if lora:
        lu = m @ bfw(w["lora_a"])           # fp32 u (saved for dB)
        sv.lu[rows] = lu
        y = y + bf16(lu) @ bfw(w["lora_b"])  # [m | bf16(u)] . [W_down ; B]
    return y


def _head(arch: Arch, W: Dict, x, emu: bool = False):
    if arch.norm == "rms":
        hf, rstd = rms_fwd(x, W["gf"], arch.rms_eps)
    else:
        hf, rstd = x, None
    if emu:
        hf = bf16(hf)
        return hf @ bfw(W["unembed"]), hf, rstd
    return hf @ W["unembed"], hf, rstd                        # :215


def _row_ce(logits_row, target):
    """row_cross_entropy, tiny_model.hpp:170-177."""
    mx = logits_row.max()
    den = np.exp(logits_row - mx).sum()
    return -(logits_row[target] - mx - math.log(den))


def generative_loss(logits, targets) -> float:
    """summed next-token CE of a window (mean applied once at the end).
    targets[i] < 0 marks a row with no next token (contributes 0 terms)."""
    s = 0.0
    for i in range(logits.shape[0]):
        if targets[i] >= 0:
            s += _row_ce(logits[i], int(targets[i]))
    return s


def forward_window(arch: Arch, W: Dict, tokens_window, l_i: int, cache: QkvCache,
                   lora: bool = True, ar=None, emu: bool = False):
    """SPEC.md:283-291 / Alg. 2 lines 3-11: positions [l_i, l_i+s) through all layers,
    attending to cached K,V [0, l_i) plus the causal window; appends Q,K,V.
    Returns (logits [s,V], final hidden [s,h])."""
    if cache.length != l_i:
        raise CacheDesync(f"cache length {cache.length} != l_i {l_i}")
    toks = np.asarray(tokens_window, dtype=np.int64)
    x = W["embed"][toks].copy()                              # tiny_model.hpp:189-190
    if emu:
        x = _bfw(x)  # rows of the bf16 embedding table (not memoised: a fresh gather)
    for n in range(arch.n_layers):
        x = _layer_forward(arch, W["layers"][n], x, l_i, cache.saved[n], lora, ar, emu)
    cache.length = l_i + len(toks)
    logits, _, _ = _head(arch, W, x, emu)
    return logits, x


def head_grad_rows(arch: Arch, W: Dict, final_hidden, targets, L: int, emu: bool = False):
    """loss_head_grad restricted to window rows (tiny_model.hpp:223-246):
    dlogits = (softmax - onehot)/(L-1) on predicting rows, 0 otherwise; -> dX through the
    (optional) final norm."""
    logits, hf, rstd = _head(arch, W, final_hidden, emu)
    dlog = np.zeros_like(logits)
    for i in range(logits.shape[0]):
        t = int(targets[i])
        if t < 0:
            continue
        row = logits[i]
        mx = row.max()
        e = np.exp(row - mx)
        dlog[i] = e / e.sum() / float(L - 1)
        dlog[i, t] -= 1.0 / float(L - 1)
    if emu:  # ce_kernel writes bf16 dlogits; dH = dlogits . U^T on the bf16 unembedding
        dh = bf16(dlog) @ bfw(W["unembed"]).T
    else:
        dh = dlog @ W["unembed"].T                            # matmul_nt :245
    if arch.norm == "rms":
        dh = rms_bwd(final_hidden, W["gf"], rstd, dh)
    return dh


def backward_window(arch: Arch, W: Dict, n: int, dY_slice, l_j: int, s_j: int,
                    cache: QkvCache, accum: KvGradAccumulator, grads: Dict,
                    state: Optional[Dict] = None, ar=None, emu: bool = False):
    """SPEC.md:292-300 / Alg. 2 lines 14-21 at layer n for rows [l_j - s_j, l_j)
    (Slice interpretation SPEC.md:333).  dY_slice is dLoss/d(layer-n output) for those rows.
    Accumulates this window's dK/dV contributions over [0, l_j) into accum (ΔKVAccum);
    rows [l_j-s_j, l_j) of accum are then final and feed dX.  LoRA grads accumulate
    into grads['a'][n], grads['b'][n] (tiny_model.hpp:280-282).
    Returns (dX slice [s_j, h], dQ [s_j, q_dim], dK contrib [l_j, kv_dim], dV contrib [l_j, kv_dim])."""
    a, b = l_j - s_j, l_j
    if state is not None:
        last = state.get((n, "next_end"))
        if last is not None and b != last:
            raise OrderingViolation(f"layer {n}: expected window ending at {last}, got {b}")
        state[(n, "next_end")] = a
    w = W["layers"][n]
    sv = cache.saved[n]
    d, Hq, Hkv = arch.head_dim, arch.n_heads, arch.n_kv_heads
    grp = Hq // Hkv
    scale = 1.0 / math.sqrt(float(d))
    rows = slice(a, b)
    dY = np.asarray(dY_slice, dtype=np.float64)
    if emu:
        return _backward_window_emu(arch, w, sv, dY, a, b, accum, grads, n)
    # --- MLP + adapter (tiny_model.hpp:276-287)
    grads["b"][n] += sv.lu[rows].T @ dY                       # :280
    d_lu = dY @ w["lora_b"].T                                 # :281
    grads["a"][n] += sv.m[rows].T @ d_lu                      # :282
    d_m = dY @ w["w_down"].T + d_lu @ w["lora_a"].T           # :283-284
    if arch.act == "relu":
        d_up = np.where(sv.m[rows] <= 0.0, 0.0, d_m)          # :285-286
        dh2 = d_up @ w["w_up"].T                              # :287
    else:
        g, u = sv.pre[rows], sv.up[rows]
        d_g = d_m * u * dsilu(g)
        d_u = d_m * silu(g)
        dh2 = d_g @ w["w_gate"].T + d_u @ w["w_up"].T
    if ar is not None:
        dh2 = ar(dh2)
    if arch.norm == "rms":
        dh2 = rms_bwd(sv.r1[rows], w["g2"], sv.rstd2[rows], dh2)
    d_r1 = dY + dh2
    # --- attention (tiny_model.hpp:289-315), query rows [a,b), keys [0,b)
    d_attn = d_r1 @ w["wo"].T                                 # :290
    dq = np.zeros((s_j, Hq * d))
    dk_c = np.zeros((b, Hkv * d))
    dv_c = np.zeros((b, Hkv * d))
    mask = np.arange(b)[None, :] <= np.arange(a, b)[:, None]
    for hq in range(Hq):
        hk = hq // grp
        qh = sv.q[rows, hq * d:(hq + 1) * d]
        kh = sv.k[:b, hk * d:(hk + 1) * d]
        vh = sv.v[:b, hk * d:(hk + 1) * d]
        sc = np.where(mask, (qh @ kh.T) * scale, -np.inf)
        p = np.exp(sc - sc.max(axis=1, keepdims=True))
        p /= p.sum(axis=1, keepdims=True)
        do = d_attn[:, hq * d:(hq + 1) * d]
        dp = do @ vh.T                                        # :300-303
        dot = np.sum(dp * p, axis=1, keepdims=True)           # :304
        ds = (dp - dot) * p                                   # :306
        dq[:, hq * d:(hq + 1) * d] = (ds @ kh) * scale        # :309
        dk_c[:, hk * d:(hk + 1) * d] += (ds.T @ qh) * scale   # :310
        dv_c[:, hk * d:(hk + 1) * d] += p.T @ do              # :311
    accum.dk[n][:b] += dk_c
    accum.dv[n][:b] += dv_c
    dk_fin = accum.dk[n][rows]                                # G_{n,j} = Slice(ΔKVAccum)
    dv_fin = accum.dv[n][rows]
    positions = np.arange(a, b)
    dq_pre, dk_pre = dq, dk_fin
    if arch.rope:
        dq_pre = rope_apply(dq, positions, Hq, d, arch.rope_theta, inverse=True)
        dk_pre = rope_apply(dk_fin, positions, Hkv, d, arch.rope_theta, inverse=True)
    dh1 = dq_pre @ w["wq"].T + dk_pre @ w["wk"].T + dv_fin @ w["wv"].T   # :317-319
    if ar is not None:
        dh1 = ar(dh1)
    if arch.norm == "rms":
        dh1 = rms_bwd(sv.x_in[rows], w["g1"], sv.rstd1[rows], dh1)
    dx = d_r1 + dh1                                           # :316
    return dx, dq, dk_c, dv_c


def _backward_window_emu(arch: Arch, w: Dict, sv: LayerSaved, dY, a: int, b: int,
                         accum: KvGradAccumulator, grads: Dict, n: int):
    """backward_window with the GPU path's bf16 points (engine.cu:backward_window):
    dycat = [bf16(dY) | bf16(dY B^T)], dm / dgu / dr1 / dO / dqkv stored bf16, P and dS bf16 as
    MMA operands inside the attention backward, fp32 dQ / dK / dV accumulation."""
    d, Hq, Hkv = arch.head_dim, arch.n_heads, arch.n_kv_heads
    grp = Hq // Hkv
    scale = 1.0 / math.sqrt(float(d))
    rows = slice(a, b)
    s_j = b - a
    Yb = bf16(dY)
    grads["b"][n] += sv.lu[rows].T @ dY                       # lora_db: fp32 u, fp32 dY
    d_lu = Yb @ bfw(w["lora_b"]).T                           # dlu GEMM (fp32 out)
    if arch.act == "relu":
        m32 = sv.m[rows]
    else:
        m32 = silu(sv.pre[rows]) * sv.up[rows]                # mlp_bwd recomputes m in fp32
    grads["a"][n] += m32.T @ d_lu
    d_m = bf16(Yb @ bfw(w["w_down"]).T + bf16(d_lu) @ bfw(w["lora_a"]).T)
    if arch.act == "relu":
        d_up = np.where(sv.m[rows] <= 0.0, 0.0, d_m)
        dh2 = d_up @ bfw(w["w_up"]).T
    else:
        g, u = sv.pre[rows], sv.up[rows]
        d_g = bf16(d_m * u * dsilu(g))
        d_u = bf16(d_m * silu(g))
        dh2 = d_g @ bfw(w["w_gate"]).T + d_u @ bfw(w["w_up"]).T
    if arch.norm == "rms":
        dh2 = rms_bwd(sv.r1[rows], w["g2"], sv.rstd2[rows], dh2)
    d_r1 = dY + dh2
    d_attn = bf16(bf16(d_r1) @ bfw(w["wo"]).T)
    dq = np.zeros((s_j, Hq * d))
    dk_c = np.zeros((b, Hkv * d))
    dv_c = np.zeros((b, Hkv * d))
    mask = np.arange(b)[None, :] <= np.arange(a, b)[:, None]
    for hq in range(Hq):
        hk = hq // grp
        qh = sv.q[rows, hq * d:(hq + 1) * d]
        kh = sv.k[:b, hk * d:(hk + 1) * d]
        vh = sv.v[:b, hk * d:(hk + 1) * d]
        sc = np.where(mask, (qh @ kh.T) * scale, -np.inf)
        mx = sc.max(axis=1, keepdims=True)
        lse = mx + np.log(np.exp(sc - mx).sum(axis=1, keepdims=True))
        p = np.exp(sc - lse)
        do = d_attn[:, hq * d:(hq + 1) * d]
        dp = do @ vh.T
        delta = np.sum(do * sv.o[rows, hq * d:(hq + 1) * d], axis=1, keepdims=True)
        dsb = bf16((dp - delta) * p)
        dq[:, hq * d:(hq + 1) * d] = (dsb @ kh) * scale
        dk_c[:, hk * d:(hk + 1) * d] += (dsb.T @ qh) * scale
        dv_c[:, hk * d:(hk + 1) * d] += bf16(p).T @ do
    accum.dk[n][:b] += dk_c
    accum.dv[n][:b] += dv_c
    dk_fin = accum.dk[n][rows]
    dv_fin = accum.dv[n][rows]
    positions = np.arange(a, b)
    dq_pre, dk_pre = dq, dk_fin
    if arch.rope:
        dq_pre = rope_apply(dq, positions, Hq, d, arch.rope_theta, inverse=True)
        dk_pre = rope_apply(dk_fin, positions, Hkv, d, arch.rope_theta, inverse=True)
    dh1 = bf16(dq_pre) @ bfw(w["wq"]).T + bf16(dk_pre) @ bfw(w["wk"]).T + bf16(dv_fin) @ bfw(w["wv"]).T
    if arch.norm == "rms":
        dh1 = rms_bwd(sv.x_in[rows], w["g1"], sv.rstd1[rows], dh1)
    dx = d_r1 + dh1
    return dx, dq, dk_c, dv_c


def lora_grads_zeros(arch: Arch) -> Dict:
    """LoraGrads::zeros, tiny_model.hpp:75-82."""
    return {"a": [np.zeros((arch.ffn, arch.lora_rank)) for _ in range(arch.n_layers)],
            "b": [np.zeros((arch.lora_rank, arch.hidden)) for _ in range(arch.n_layers)]}


# ---------------------------------------------------------------------------
# Full-sequence oracle = a single window (SPEC.md:289,299 degenerate partitions)
# ---------------------------------------------------------------------------

def forward_full(arch: Arch, W: Dict, tokens, ar=None, emu: bool = False):
    """tiny_model.hpp:181-221."""
    L = len(tokens)
    if L < 1:
        raise ValueError("forward_full: empty sequence")     # :183
    cache = QkvCache(arch, L)
    logits, final = forward_window(arch, W, tokens, 0, cache, ar=ar, emu=emu)
    targets = np.concatenate([np.asarray(tokens[1:], dtype=np.int64), [-1]])
    loss = generative_loss(logits, targets) / float(L - 1) if L > 1 else 0.0
    return {"tokens": np.asarray(tokens), "cache": cache, "logits": logits,
            "final_hidden": final, "loss": loss, "emu": emu}


def backward_full(arch: Arch, W: Dict, tr, windows: Optional[List[int]] = None, ar=None):
    """tiny_model.hpp:259-327, optionally executed as token-level backward windows
    (sizes listed in reverse traversal order; default one window per layer)."""
    tokens = tr["tokens"]
    L = len(tokens)
    targets = np.concatenate([tokens[1:], [-1]])
    emu = tr.get("emu", False)
    dy = head_grad_rows(arch, W, tr["final_hidden"], targets, L, emu) if L > 1 else \
        np.zeros((L, arch.hidden))
    grads = lora_grads_zeros(arch)
    accum = KvGradAccumulator(arch, L)
    layers = [None] * arch.n_layers
    for n in range(arch.n_layers - 1, -1, -1):
        dx = np.zeros((L, arch.hidden))
        dq_all = np.zeros((L, arch.q_dim))
        lj = L
        for s in (windows or [L]):
            s = min(s, lj)
            if s <= 0:
                break
            dxs, dq, _, _ = backward_window(arch, W, n, dy[lj - s:lj], lj, s, tr["cache"],
                                            accum, grads, ar=ar, emu=emu)
            dx[lj - s:lj] = dxs
            dq_all[lj - s:lj] = dq
            lj -= s
        assert lj == 0, "windows must partition [0, L)"
        layers[n] = {"dk": accum.dk[n], "dv": accum.dv[n], "dx": dx, "dq": dq_all}
        dy = dx
    if ar is not None:  # TP: dB partial sums (folded LoRA), reduced once per mini-batch
        grads["b"] = [ar(g) for g in grads["b"]]
    return {"loss": tr["loss"], "grads": grads, "layers": layers}


# ---------------------------------------------------------------------------
# Metrics (matrix.hpp:121-139, tiny_model.hpp:85-92)
# ---------------------------------------------------------------------------

def max_rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(1e-30, float(np.max(np.abs(b))) if b.size else 0.0)
    m = float(np.max(np.abs(a - b))) if a.size else 0.0
    return m / max(1.0, scale)


def rel_err(a: float, b: float) -> float:
    return abs(a - b) / max(1.0, abs(b))


def scaled_err(a, b) -> float:
    """Scale-normalised error max|a-b| / max|b| (SURVEY.md §7 hard part (e))."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(1e-30, float(np.max(np.abs(b)))))


def max_grad_rel_err(x: Dict, ref: Dict) -> float:
    m = 0.0
    for l in range(len(ref["a"])):
        m = max(m, max_rel_err(x["a"][l], ref["a"][l]), max_rel_err(x["b"][l], ref["b"][l]))
    return m


# ---------------------------------------------------------------------------
# Adam (PAPER.md:432 -- hyperparameters unspecified by the reference;
# ours are declared in DESIGN.md)
# ---------------------------------------------------------------------------

@dataclass
class AdamConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


def adam_step(p, g, m, v, t: int, cfg: AdamConfig):
    """Kingma & Ba Adam with bias correction; t is the 1-based step count."""
    m[:] = cfg.beta1 * m + (1.0 - cfg.beta1) * g
    v[:] = cfg.beta2 * v + (1.0 - cfg.beta2) * g * g
    mhat = m / (1.0 - cfg.beta1 ** t)
    vhat = v / (1.0 - cfg.beta2 ** t)
    p[:] = p - cfg.lr * mhat / (np.sqrt(vhat) + cfg.eps)
    return p
