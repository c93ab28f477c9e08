"""GPU parity of the co-serving step (cs_step through the C ABI) against the CPU oracle.

* reference arch (BASELINE config 1: 2 layers, h=256, 4 heads, r=8, V=64; 16 decode rows +
  64 finetuning tokens): weights from TinyModel::init (bit-exact restatement), FT loss / LoRA
  grads / ΔKVAccum / dX vs the reference's forward_full + backward_full (tiny_model.hpp:181-327),
  inference logits vs the window restatement.
* LLaMA/Qwen arch (RMSNorm, RoPE, SwiGLU, GQA, QKV bias) vs the numpy oracle.
Two references per quantity (north_star: bf16 with fp32 accumulate, rel <= 1e-2):
* the bf16 rounding-point oracle (coserve_oracle emu=True: the same arithmetic with bf16 at
  every point where the GPU stores or feeds bf16) -- the GPU must match it to scale-normalised
  max|a-b|/max|b| <= 1e-2 (EMU_TOL) for logits, loss, LoRA grads of every layer, dK/dV/dX.
  Exception, by measurement: where the emu oracle drifts from ITSELF by more than 1e-2 under
  fp32-level (3e-7) activation noise (O.emu_sensitivity -- the reference arch's ReLU backward
  mask, tiny_model.hpp:285-286, makes its deep dX / layer-0 grads chaotic at bf16), the bound
  is 2x that self-drift: no bf16 implementation can sit closer to another;
* the f64 oracle (the reference's arithmetic) -- bounded by the bf16 storage floor
  (FLOOR_TOP / FLOOR_DEEP) that the emu oracle itself shows against f64, and the reference's
  own metric max_rel_err (matrix.hpp:127-135) < 1e-2.
Set CS_PARITY_LOG=path to append every measured error to a JSON-lines report.
"""
import json
import os

import numpy as np
import pytest

from oracle import coserve_oracle as O
from paper_2402_18789_b200.engine import (Engine, Seg, arch_config, SEG_DECODE, SEG_PREFILL,
                                          SEG_FT_FWD, FT_FORWARD, FT_BACKWARD)
from paper_2402_18789_b200 import _lib

pytestmark = pytest.mark.gpu

TOL = 1e-2
EMU_TOL = 1e-2
# where the emu oracle's own fp32-noise drift exceeds EMU_TOL the bound is DRIFT_FACTOR x that
# drift: GPU-vs-emu and noisy-emu-vs-emu are the same statistic (two independent draws of the
# bf16 rounding noise, max over the same elements), 2x covers the spread of that max
DRIFT_FACTOR = 2.0
# Scale-normalised (max|a-b|/max|b|) bounds against the f64 oracle: the bf16 storage floor
# (emu oracle vs f64) is 0.5% (top layer grads), 2.7-3.4% (bottom layer grads, after two
# attention backwards) and 2-6% (dK/dV/dX of layer 1); ~1.5x headroom over that floor.
FLOOR_TOP, FLOOR_DEEP = 0.02, 0.08


class Pages:
    def __init__(self, n):
        self.free = list(range(n - 1, -1, -1))

    def take(self, k):
        return [self.free.pop() for _ in range(k)]


def _log(rec):
    path = os.environ.get("CS_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


class Sensitivity:
    """Lazily computed O.emu_sensitivity of one (arch, weights, tokens) case."""

    def __init__(self, arch, W, toks, clean=None, trials=3):
        self.args, self.kw, self.val = (arch, W, toks), {"clean": clean, "trials": trials}, None

    def __getitem__(self, q):
        if self.val is None:
            self.val = O.emu_sensitivity(*self.args, **self.kw)
        return self.val.get(q, 0.0)


def gate(test, name, gpu, emu_ref, f64_ref, floor, sens=None, emu_tol=EMU_TOL):
    """GPU vs the bf16 rounding-point oracle at emu_tol (north_star rel <= 1e-2; or 2x the
    oracle's own measured fp32-noise drift where that exceeds it) and vs f64 under the bf16
    storage floor; the reference's max_rel_err also < 1e-2.  An all-zero gradient scores 1.0
    on both scale-normalised checks, so these gates can fail."""
    e_emu = O.scaled_err(gpu, emu_ref)
    e_f64 = O.scaled_err(gpu, f64_ref)
    e_mre = O.max_rel_err(gpu, f64_ref)
    e_floor = O.scaled_err(emu_ref, f64_ref)
    tol = emu_tol
    drift = None
    if e_emu > emu_tol and sens is not None:
        drift = sens[name]
        tol = max(emu_tol, DRIFT_FACTOR * drift)
    _log({"test": test, "q": name, "gpu_vs_emu": e_emu, "gpu_vs_f64": e_f64,
          "emu_vs_f64": e_floor, "max_rel_err": e_mre, "emu_self_drift": drift, "tol": tol})
    assert e_emu <= tol, (name, "gpu vs bf16-emulated oracle", e_emu, "emu self-drift", drift)
    assert e_f64 < floor, (name, "gpu vs f64 oracle", e_f64, "emu floor", e_floor)
    assert e_mre < TOL, (name, "max_rel_err", e_mre)
    return e_emu


def noisy_emu_drift(arch, W, toks, pos, cache_n, clean_logits, rng, amp=3e-7):
    """The same inference row through the emu oracle with fp32-level activation noise (its
    own cache, fed the same tokens): how far a bf16 evaluation drifts from itself."""
    O._NOISE = (rng, amp)
    try:
        ln, _ = O.forward_window(arch, W, toks, pos, cache_n, lora=False, emu=True)
    finally:
        O._NOISE = None
    return O.scaled_err(ln[-1], clean_logits[-1])


def logit_emu_tol(drift):
    """Logit rows are max-normalised over a small vocabulary: a few bf16 flips of the final
    hidden state move the max entry by ~0.5-1%; tolerance = max(1e-2, DRIFT_FACTOR x the largest
    self-drift of the same rows (the GPU is one more independent draw of that noise))."""
    return max(EMU_TOL, DRIFT_FACTOR * max(drift)) if drift else EMU_TOL


def oracles(arch, W, toks):
    tr = O.forward_full(arch, W, toks)
    bw = O.backward_full(arch, W, tr)
    te = O.forward_full(arch, W, toks, emu=True)
    be = O.backward_full(arch, W, te)
    return tr, bw, te, be


def gate_grads(test, arch, eng, bw, be, kvg, dys, kv_layers=(1,), floor_deep=FLOOR_DEEP, sens=None):
    for l in range(arch.n_layers):
        ga, gb = eng.lora_grads(l)
        floor = FLOOR_TOP if l == arch.n_layers - 1 else floor_deep
        gate(test, f"dA{l}", ga, be["grads"]["a"][l], bw["grads"]["a"][l], floor, sens)
        gate(test, f"dB{l}", gb, be["grads"]["b"][l], bw["grads"]["b"][l], floor, sens)
    for n in kv_layers:
        dk, dv = kvg[n]
        gate(test, f"dK{n}", dk, be["layers"][n]["dk"], bw["layers"][n]["dk"], floor_deep, sens)
        gate(test, f"dV{n}", dv, be["layers"][n]["dv"], bw["layers"][n]["dv"], floor_deep, sens)
        gate(test, f"dX{n}", dys[n], be["layers"][n]["dx"], bw["layers"][n]["dx"], floor_deep, sens)


def gate_loss(test, loss, tr, te):
    e_emu, e_f64 = O.rel_err(loss, te["loss"]), O.rel_err(loss, tr["loss"])
    _log({"test": test, "q": "loss", "gpu_vs_emu": e_emu, "gpu_vs_f64": e_f64})
    assert e_emu < EMU_TOL and e_f64 < TOL, (loss, te["loss"], tr["loss"])


def _run_coserve(arch, W, ft_tokens, fwd_windows, bwd_windows, n_inf=16, seed=7, P=16,
                 check_logits=True, logit_tol=TOL, test="coserve"):
    """Drive the engine through prefill -> mixed decode+FT-forward -> FT backward windows,
    mirroring each inference request on the f64 and the bf16-emulated oracle.  Returns the
    engine, the accumulated FT loss sum, ΔKVAccum and dX per layer, and the largest
    inference-logit error against f64."""
    cfg = arch_config(arch, page_size=P, n_pages=256, max_tokens=512, max_ft_len=len(ft_tokens),
                      max_segments=64)
    eng = Engine(cfg)
    eng.load_weights(W)
    rng = O.Rng(seed)
    pages = Pages(256)
    L = len(ft_tokens)
    ft_pages = pages.take((L + P - 1) // P)
    reqs = []
    for i in range(n_inf):
        plen = rng.uniform_int(3, 20)
        toks = [rng.uniform_int(0, arch.vocab - 1) for _ in range(plen)]
        reqs.append({"tokens": toks, "pages": pages.take((plen + 8 + P - 1) // P),
                     "cache": O.QkvCache(arch, plen + 8), "cache_e": O.QkvCache(arch, plen + 8),
                     "cache_n": O.QkvCache(arch, plen + 8), "len": 0})
    diffs, ediffs, drift = [], [], []
    noise_rng = np.random.default_rng(99)

    def check(i, r, toks, pos, out):
        lg, _ = O.forward_window(arch, W, toks, pos, r["cache"], lora=False)
        le, _ = O.forward_window(arch, W, toks, pos, r["cache_e"], lora=False, emu=True)
        diffs.append(O.scaled_err(out["logits"][i], lg[-1]))
        ediffs.append(O.scaled_err(out["logits"][i], le[-1]))
        drift.append(noisy_emu_drift(arch, W, toks, pos, r["cache_n"], le, noise_rng))

    # step 1: prefill every prompt (sampled)
    segs = [Seg(SEG_PREFILL, r["tokens"], 0, r["pages"], sample=True) for r in reqs]
    out = eng.step(segs, want_logits=True)
    for i, r in enumerate(reqs):
        check(i, r, r["tokens"], 0, out)
        r["len"] = len(r["tokens"])
        assert out["next_tokens"][i] == int(np.argmax(out["logits"][i]))
    # forward windows, each fused with one decode row per request
    loss_sum = 0.0
    l = 0
    for s in fwd_windows:
        segs = []
        for r in reqs:
            t = rng.uniform_int(0, arch.vocab - 1)
            segs.append(Seg(SEG_DECODE, [t], r["len"], r["pages"], sample=True))
            r["pending"] = t
        segs.append(Seg(SEG_FT_FWD, ft_tokens[l:l + s], l, ft_pages, adapter=True))
        targets = [ft_tokens[i + 1] if i + 1 < L else -1 for i in range(l, l + s)]
        out = eng.step(segs, ft={"phase": FT_FORWARD, "seq_len": L, "l": l, "s": s,
                                 "targets": targets}, want_logits=True)
        loss_sum += out["loss_sum"]
        for i, r in enumerate(reqs):
            check(i, r, [r["pending"]], r["len"], out)
            r["len"] += 1
        l += s
    # backward windows (layer N-1 .. 0), alone in the batch
    kvgrads = {}
    dys = {}
    for n in range(arch.n_layers - 1, -1, -1):
        lj = L
        for s in bwd_windows:
            s = min(s, lj)
            eng.step([], ft={"phase": FT_BACKWARD, "seq_len": L, "l": lj, "s": s, "layer": n,
                             "pages": ft_pages})
            lj -= s
            if lj == 0:
                break
        if n > 0:
            kvgrads[n] = eng.kvgrad(L)
            dys[n] = eng.read_dy(L)
    tol = logit_emu_tol(drift)
    _log({"test": test, "q": "inference_logits", "gpu_vs_f64": max(diffs),
          "gpu_vs_emu": max(ediffs), "emu_self_drift": max(drift), "tol": tol})
    if check_logits:
        assert max(diffs) < logit_tol, max(diffs)
        assert max(ediffs) <= tol, ("logits vs bf16-emulated oracle", max(ediffs), max(drift))
    return eng, loss_sum, kvgrads, dys, max(diffs)


def test_reference_tiny_config_parity():
    """BASELINE config 1 against the reference's arithmetic (f64) and the bf16-emulated oracle."""
    arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
    W = O.init_tiny(arch, 1)
    toks = list(O.Rng(42).uniform_int(0, 63, 64))
    tr, bw, te, be = oracles(arch, W, toks)
    eng, loss_sum, kvg, dys, dmax = _run_coserve(arch, W, toks, [64], [64], test="tiny_cfg1")
    loss = loss_sum / 63.0
    assert abs(loss - 4.1809416937891104) < 1e-2 * 4.18  # SURVEY Appendix A (cfg B)
    gate_loss("tiny_cfg1", loss, tr, te)
    gate_grads("tiny_cfg1", arch, eng, bw, be, kvg, dys, sens=Sensitivity(arch, W, toks, clean=be))


@pytest.mark.parametrize("fwd,bwd", [([20, 30, 14], [24, 24, 16]), ([1, 63], [7, 57])])
def test_token_level_windows_match_full_sequence(fwd, bwd):
    """Alg. 2 equivalence on the GPU: any window partition gives the full-sequence loss, LoRA
    grads, ΔKVAccum and dX (gated against the full-sequence oracles, scale-normalised)."""
    arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
    W = O.init_tiny(arch, 1)
    toks = list(O.Rng(42).uniform_int(0, 63, 64))
    tr, bw, te, be = oracles(arch, W, toks)
    eng, loss_sum, kvg, dys, _ = _run_coserve(arch, W, toks, fwd, bwd, n_inf=4,
                                              test=f"windows_{fwd}_{bwd}")
    gate_loss("windows", loss_sum / 63.0, tr, te)
    gate_grads(f"windows_{fwd}_{bwd}", arch, eng, bw, be, kvg, dys, sens=Sensitivity(arch, W, toks, clean=be))


LLAMA3 = O.Arch(n_layers=3, hidden=256, n_heads=4, n_kv_heads=2, head_dim=64, ffn=512,
                vocab=128, lora_rank=16, norm="rms", act="swiglu", rope=True, qkv_bias=True,
                rope_theta=10000.0)


def test_llama_arch_parity():
    arch = LLAMA3
    W = O.init_general(arch, 3)
    toks = list(np.random.default_rng(5).integers(0, arch.vocab, 100))
    tr, bw, te, be = oracles(arch, W, toks)
    # RMSNorm/RoPE/SwiGLU in bf16: inference logits sit at ~2% of max|logit| vs f64 (bf16 floor)
    eng, loss_sum, kvg, dys, _ = _run_coserve(arch, W, toks, [40, 60], [30, 30, 40], n_inf=5,
                                              logit_tol=0.04, test="llama3")
    gate_loss("llama3", loss_sum / 99.0, tr, te)
    gate_grads("llama3", arch, eng, bw, be, kvg, dys, kv_layers=(1, 2), sens=Sensitivity(arch, W, toks, clean=be))


def test_adam_update_matches_oracle():
    """cs_adam_step == oracle Adam applied to the engine's own gradients;
    and the update direction agrees with the f64 reference gradients where they are
    resolvable above the bf16 floor."""
    arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
    W = O.init_tiny(arch, 1)
    toks = list(O.Rng(42).uniform_int(0, 63, 64))
    tr = O.forward_full(arch, W, toks)
    bw = O.backward_full(arch, W, tr)
    eng, _, _, _, _ = _run_coserve(arch, W, toks, [64], [64], n_inf=2)
    cfg = O.AdamConfig(lr=1e-3)
    grads = [eng.lora_grads(l) for l in range(arch.n_layers)]
    before = [eng.lora(l) for l in range(arch.n_layers)]
    eng.adam_step(cfg.lr, cfg.beta1, cfg.beta2, cfg.eps)
    for l in range(arch.n_layers):
        after = eng.lora(l)
        for i, key in enumerate(("lora_a", "lora_b")):
            p = before[l][i].copy()
            g = grads[l][i]
            O.adam_step(p, g, np.zeros_like(p), np.zeros_like(p), 1, cfg)
            assert np.abs(after[i] - p).max() < 1e-6 + 1e-5 * np.abs(p).max()
            ref_g = bw["grads"]["a" if i == 0 else "b"][l]
            big = np.abs(ref_g) > 0.1 * np.abs(ref_g).max()
            upd = after[i] - before[l][i]
            assert (np.sign(upd[big]) == -np.sign(ref_g[big])).mean() > 0.99
    with pytest.raises(_lib.OrderingViolation):  # second Adam without a new backward pass
        eng.adam_step()


def test_errors_follow_reference_conventions():
    arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
    W = O.init_tiny(arch, 1)
    eng = Engine(arch_config(arch, n_pages=32, max_tokens=128, max_ft_len=64))
    eng.load_weights(W)
    toks = list(O.Rng(42).uniform_int(0, 63, 64))
    pages = list(range(4))
    with pytest.raises(_lib.CacheDesync):  # SPEC.md:291 l_i=2 on an empty cache
        eng.step([Seg(SEG_FT_FWD, toks[2:4], 2, pages, adapter=True)],
                 ft={"phase": FT_FORWARD, "seq_len": 64, "l": 2, "s": 2, "targets": [1, 2]})
    with pytest.raises(_lib.OrderingViolation):  # backward before forward complete
        eng.step([], ft={"phase": FT_BACKWARD, "seq_len": 64, "l": 64, "s": 8, "layer": 1,
                         "pages": pages})
    eng.step([Seg(SEG_FT_FWD, toks, 0, pages, adapter=True)],
             ft={"phase": FT_FORWARD, "seq_len": 64, "l": 0, "s": 64,
                 "targets": toks[1:] + [-1]})
    with pytest.raises(_lib.OrderingViolation):  # wrong layer first
        eng.step([], ft={"phase": FT_BACKWARD, "seq_len": 64, "l": 64, "s": 8, "layer": 0,
                         "pages": pages})
    with pytest.raises(ValueError):  # token id out of range
        eng.step([Seg(SEG_PREFILL, [999], 0, [5])])
    with pytest.raises(ValueError):  # page table does not cover the context
        eng.step([Seg(SEG_PREFILL, list(range(20)), 0, [5])])


ARCH_D128 = O.Arch(n_layers=2, hidden=512, n_heads=4, n_kv_heads=2, head_dim=128, ffn=512,
                   vocab=128, lora_rank=8, norm="rms", act="swiglu", rope=True, qkv_bias=False,
                   rope_theta=10000.0)


@pytest.mark.parametrize("tc", ["1", "0"])
def test_d128_tcgen05_attention_parity(tc, monkeypatch):
    """head_dim 128: prefill / FT-window rows run on the tcgen05 attention kernels (CS_ATTN_TC=1:
    forward attn_fwd_tc2, backward the fused dK/dV/dQ kernel) or the mma.sync kernels (0);
    contexts span several 128-key tiles and a window boundary that is not tile aligned."""
    monkeypatch.setenv("CS_ATTN_TC", tc)
    arch = ARCH_D128
    W = O.init_general(arch, 7)
    toks = list(np.random.default_rng(9).integers(0, arch.vocab, 300))
    tr, bw, te, be = oracles(arch, W, toks)
    t = f"d128_tc{tc}"
    eng, loss_sum, kvg, dys, dmax = _run_coserve(arch, W, toks, [100, 200], [150, 150], n_inf=5,
                                                 logit_tol=0.04, test=t)
    gate_loss(t, loss_sum / 299.0, tr, te)
    gate_grads(t, arch, eng, bw, be, kvg, dys, sens=Sensitivity(arch, W, toks, clean=be))


def test_reference_arch_d128_vs_live_reference():
    """The reference's own arch at head_dim 128 (hidden 512, 4 heads, MHA, ReLU, no norm):
    the tcgen05 attention forward / backward kernels against tiny_model.hpp:120-151,259-327
    compiled unmodified (oracle/_ref) -- loss, LoRA grads, dK/dV/dX of layer 1 -- and against
    the bf16-emulated oracle at 1e-2."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    arch = O.Arch.reference(depth=2, hidden=512, heads=4, vocab=64, rank=8)
    m = R.RefTinyModel(depth=2, hidden=512, heads=4, ffn_mult=4, vocab=64, rank=8, seed=1)
    W = m.weights()
    toks = [int(t) for t in O.Rng(42).uniform_int(0, 63, 256)]
    ref = m.forward_backward(toks)
    te = O.forward_full(arch, W, toks, emu=True)
    be = O.backward_full(arch, W, te)
    bw = {"grads": {"a": list(ref["grad_a"]), "b": list(ref["grad_b"])},
          "layers": [{"dk": ref["dk"][n], "dv": ref["dv"][n], "dx": ref["dx"][n]}
                     for n in range(2)]}
    tr = {"loss": ref["loss"]}
    eng, loss_sum, kvg, dys, _ = _run_coserve(arch, W, toks, [100, 156], [128, 128], n_inf=6,
                                              logit_tol=0.04, test="ref_d128")
    gate_loss("ref_d128", loss_sum / 255.0, tr, te)
    gate_grads("ref_d128", arch, eng, bw, be, kvg, dys, sens=Sensitivity(arch, W, toks, clean=be))


ARCH_GQA4 = O.Arch(n_layers=2, hidden=512, n_heads=4, n_kv_heads=1, head_dim=128, ffn=512,
                   vocab=128, lora_rank=8, norm="rms", act="swiglu", rope=True, qkv_bias=False,
                   rope_theta=10000.0)


@pytest.mark.parametrize("dec", ["1", "0"])
def test_decode_attention_kernel_parity(dec, monkeypatch):
    """Decode rows (q_len * group <= 16) on the HBM-bound paged decode kernel (CS_ATTN_DEC=1)
    or the mma.sync tile kernel (0), LLaMA-8B head geometry (group 4, d=128): contexts from 1
    to 700 keys (split across CTAs and merged by LSE), ragged pages, multi-row (q_len 3)
    segments, all against the oracle's window forward."""
    monkeypatch.setenv("CS_ATTN_DEC", dec)
    arch = ARCH_GQA4
    W = O.init_general(arch, 11)
    P = 16
    eng = Engine(arch_config(arch, page_size=P, n_pages=512, max_tokens=2048, max_ft_len=16,
                             max_segments=64))
    eng.load_weights(W)
    rng = np.random.default_rng(3)
    pages = Pages(512)
    reqs = []
    for plen in (1, 3, 5, 37, 300, 700, 129):
        toks = [int(t) for t in rng.integers(0, arch.vocab, plen)]
        pg = pages.take((plen + 8 + P - 1) // P)
        pg = pg[::-1]  # non-monotone page ids
        reqs.append({"tokens": toks, "pages": pg, "cache": O.QkvCache(arch, plen + 8),
                     "cache_e": O.QkvCache(arch, plen + 8), "cache_n": O.QkvCache(arch, plen + 8),
                     "len": 0})
    out = eng.step([Seg(SEG_PREFILL, r["tokens"], 0, r["pages"], sample=True) for r in reqs],
                   want_logits=True)
    diffs, ediffs, drift = [], [], []
    nrng = np.random.default_rng(98)

    def check(i, r, toks, pos):
        lg, _ = O.forward_window(arch, W, toks, pos, r["cache"], lora=False)
        le, _ = O.forward_window(arch, W, toks, pos, r["cache_e"], lora=False, emu=True)
        diffs.append(O.scaled_err(out["logits"][i], lg[-1]))
        ediffs.append(O.scaled_err(out["logits"][i], le[-1]))
        drift.append(noisy_emu_drift(arch, W, toks, pos, r["cache_n"], le, nrng))

    for i, r in enumerate(reqs):
        check(i, r, r["tokens"], 0)
        r["len"] = len(r["tokens"])
    for _ in range(3):
        segs = []
        for r in reqs:
            r["pending"] = int(rng.integers(0, arch.vocab))
            segs.append(Seg(SEG_DECODE, [r["pending"]], r["len"], r["pages"], sample=True))
        out = eng.step(segs, want_logits=True)
        for i, r in enumerate(reqs):
            check(i, r, [r["pending"]], r["len"])
            r["len"] += 1
    tol = logit_emu_tol(drift)
    _log({"test": f"decode_{dec}", "q": "logits", "gpu_vs_f64": max(diffs), "gpu_vs_emu": max(ediffs),
          "emu_self_drift": max(drift), "tol": tol})
    assert max(diffs) < 0.04, max(diffs)
    assert max(ediffs) <= tol, (max(ediffs), max(drift))
    eng.close()


def test_alloc_audit_no_frozen_weight_gradients():
    """Matrix::alloc_hook analogue (matrix.hpp:16-25): a full finetuning pass (forward windows,
    backward windows through every layer, Adam) allocates no device memory, and the only
    model-sized fp32 buffers are the LoRA state (graph pruning: frozen dW is never formed)."""
    arch = O.Arch(n_layers=3, hidden=256, n_heads=4, n_kv_heads=2, head_dim=64, ffn=512,
                  vocab=128, lora_rank=16, norm="rms", act="swiglu", rope=True, qkv_bias=True,
                  rope_theta=10000.0)
    W = O.init_general(arch, 3)
    toks = list(np.random.default_rng(5).integers(0, arch.vocab, 100))
    # capacities chosen so no activation buffer is coincidentally weight-sized
    cfg = arch_config(arch, page_size=16, n_pages=256, max_tokens=200, max_ft_len=len(toks),
                      max_segments=64)
    eng = Engine(cfg)
    eng.load_weights(W)
    recs0, tr0 = eng.alloc_audit()
    _run_coserve_on(eng, arch, W, toks, [40, 60], [30, 30, 40])
    eng.adam_step()
    recs1, tr1 = eng.alloc_audit()
    assert tr1 == tr0 and recs1 == recs0          # nothing allocated by steps / Adam
    names = {n for n, _, _ in recs1}
    assert {"gA", "gB", "dk_acc", "dv_acc"} <= names
    # fp32 buffers whose size does not move with the engine's capacities (tokens, FT length,
    # pages, segments) are model-sized: they must be exactly the LoRA master/grad/Adam state, the norm
    # gains and biases, and the fixed split-KV scratch -- no frozen-weight gradient
    cfg2 = arch_config(arch, page_size=16, n_pages=300, max_tokens=300, max_ft_len=120,
                       max_segments=80)
    eng2 = Engine(cfg2)
    recs2, _ = eng2.alloc_audit()
    eng2.close()
    size1 = {n: (el, b) for n, el, b in recs1}
    model_sized = {n for n, el, b in recs2 if b == 4 and size1.get(n) == (el, b)}
    allowed = {"gf", "bqkv", "g1", "g2", "loraA", "loraB", "gA", "gB", "mA", "vA", "mB", "vB",
               "part_o", "part_lse", "part_o_tc", "part_lse_tc", "tp_sync", "tp_stage", "ipc_flags"}
    assert model_sized <= allowed, model_sized - allowed
    NL, f, r, h = arch.n_layers, arch.ffn, arch.lora_rank, arch.hidden
    assert size1["gA"][0] == NL * f * r and size1["gB"][0] == NL * r * h
    eng.close()


def _run_coserve_on(eng, arch, W, toks, fwd, bwd):
    from paper_2402_18789_b200.engine import Seg as S
    L = len(toks)
    pages = list(range(200, 200 + (L + 15) // 16))
    l = 0
    for s in fwd:
        eng.step([S(SEG_FT_FWD, toks[l:l + s], l, pages, adapter=True)],
                 ft={"phase": FT_FORWARD, "seq_len": L, "l": l, "s": s,
                     "targets": [toks[i + 1] if i + 1 < L else -1 for i in range(l, l + s)]})
        l += s
    for n in range(arch.n_layers - 1, -1, -1):
        lj = L
        for s in bwd:
            s = min(s, lj)
            eng.step([], ft={"phase": FT_BACKWARD, "seq_len": L, "l": lj, "s": s, "layer": n,
                             "pages": pages})
            lj -= s
            if lj == 0:
                break


def test_tc_attention_split_kv_parity():
    """Prefill chunks at long context on the tcgen05 attention kernel: few work items, so the
    key ranges are split into parts merged by the LSE combine (flash-decoding style)."""
    arch = ARCH_GQA4
    W = O.init_general(arch, 13)
    P = 16
    L = 2600
    eng = Engine(arch_config(arch, page_size=P, n_pages=256, max_tokens=1024, max_ft_len=16,
                             max_segments=8))
    eng.load_weights(W)
    toks = [int(t) for t in np.random.default_rng(21).integers(0, arch.vocab, L)]
    pages = list(range(200))[::-1][: (L + 8 + P - 1) // P]
    cache = O.QkvCache(arch, L + 8)
    cache_e = O.QkvCache(arch, L + 8)
    cache_n = O.QkvCache(arch, L + 8)
    diffs, ediffs, drift = [], [], []
    nrng = np.random.default_rng(97)
    for c0 in range(0, L, 512):
        chunk = toks[c0:c0 + 512]
        out = eng.step([Seg(SEG_PREFILL, chunk, c0, pages, sample=True)], want_logits=True)
        lg, _ = O.forward_window(arch, W, chunk, c0, cache, lora=False)
        le, _ = O.forward_window(arch, W, chunk, c0, cache_e, lora=False, emu=True)
        diffs.append(O.scaled_err(out["logits"][0], lg[-1]))
        ediffs.append(O.scaled_err(out["logits"][0], le[-1]))
        drift.append(noisy_emu_drift(arch, W, chunk, c0, cache_n, le, nrng))
    tol = logit_emu_tol(drift)
    _log({"test": "split_kv", "q": "logits", "gpu_vs_f64": max(diffs), "gpu_vs_emu": max(ediffs),
          "emu_self_drift": max(drift), "tol": tol})
    assert max(diffs) < 0.04, diffs
    assert max(ediffs) <= tol, (ediffs, drift)
    eng.close()


ARCH_QWEN5 = O.Arch(n_layers=2, hidden=640, n_heads=10, n_kv_heads=2, head_dim=128, ffn=512,
                    vocab=128, lora_rank=16, norm="rms", act="swiglu", rope=True, qkv_bias=True,
                    rope_theta=1000000.0)


def test_qwen_geometry_gqa5_parity():
    """Qwen-2.5 head geometry (40 q / 8 kv heads -> GQA group 5, d=128,
    QKV bias, rope theta 1e6) scaled down: a group that does not divide the 128-row packed
    query tiles (25 positions x 5 heads + 3 pad rows) on the tcgen05 forward, the decode kernel
    (5 rows of the m16 tile) and the backward (group 5 does not divide 64 -> the tile kernel)."""
    arch = ARCH_QWEN5
    W = O.init_general(arch, 17)
    toks = list(np.random.default_rng(23).integers(0, arch.vocab, 300))
    tr, bw, te, be = oracles(arch, W, toks)
    eng, loss_sum, kvg, dys, _ = _run_coserve(arch, W, toks, [100, 200], [150, 150], n_inf=5,
                                              logit_tol=0.04, test="qwen_gqa5")
    gate_loss("qwen_gqa5", loss_sum / 299.0, tr, te)
    gate_grads("qwen_gqa5", arch, eng, bw, be, kvg, dys, sens=Sensitivity(arch, W, toks, clean=be))
    eng.close()
