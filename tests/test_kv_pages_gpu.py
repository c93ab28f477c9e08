"""KV/page indexing parity (north_star: "KV/page indexing bit-exact").

The paged K/V pools are read back through cs_read_kv (include/coserve_cuda.h) and compared
slot by slot with what the oracle says each position's K/V row is:

* bit-exact: the reference arch (no norm, no RoPE) with layer-0 W_k / W_v set to permutation
  matrices, so every K/V row is exactly a permuted bf16 embedding row (one non-zero product per
  output: the fp32 GEMM accumulation is exact and the bf16 store is lossless).  Any misplaced
  row, wrong page, wrong slot-in-page, stale write or column permutation shows up as a bit
  difference.  Ragged prompts on non-monotone pages, chunked prefill continuing mid-page, decode
  rows crossing page boundaries and a finetuning window in its own pages all write in one
  engine; pages nobody owns must be untouched.
* LLaMA arch (RMSNorm, RoPE, GQA): every slot within two bf16 ulps (of the row's scale) of the
  bf16-emulated oracle's K/V, and each stored row closest to its own position's oracle row.
"""
import numpy as np
import pytest

from oracle import coserve_oracle as O
from paper_2402_18789_b200.engine import (Engine, Seg, arch_config, SEG_DECODE, SEG_PREFILL,
                                          SEG_FT_FWD, FT_FORWARD)

pytestmark = pytest.mark.gpu

P = 16


def _perm_weights(arch, seed):
    W = O.init_tiny(arch, 1)
    rng = np.random.default_rng(seed)
    h = arch.hidden
    for key in ("wk", "wv"):
        perm = rng.permutation(h)
        M = np.zeros((h, h))
        M[np.arange(h), perm] = 1.0       # out[:, perm[i]] = x[:, i]
        W["layers"][0][key] = M
    return W


def _expected_kv(W, toks, key):
    xb = O.bf16(W["embed"][np.asarray(toks)])
    return xb @ W["layers"][0][key]


def test_kv_pages_bit_exact_reference_arch():
    arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
    W = _perm_weights(arch, 5)
    n_pages = 96
    eng = Engine(arch_config(arch, page_size=P, n_pages=n_pages, max_tokens=256, max_ft_len=96,
                             max_segments=32))
    eng.load_weights(W)
    rng = np.random.default_rng(11)
    free = list(rng.permutation(n_pages))
    reqs = []
    for plen in (1, 5, 16, 17, 33, 47):
        toks = [int(t) for t in rng.integers(0, arch.vocab, plen)]
        pages = [int(free.pop()) for _ in range((plen + 40 + P - 1) // P)]
        reqs.append({"toks": toks, "pages": pages, "len": 0})
    untouched = [int(free.pop()) for _ in range(6)]
    before = eng.read_kv(0, untouched, len(untouched) * P)
    # step 1: prefill, the 47-token prompt split: first 20 tokens now, the rest next step
    segs = []
    for r in reqs:
        n = 20 if len(r["toks"]) == 47 else len(r["toks"])
        segs.append(Seg(SEG_PREFILL, r["toks"][:n], 0, r["pages"], sample=True))
        r["len"] = n
    eng.step(segs)
    # step 2: the chunk continuing mid-page + one decode row for every other request
    segs = []
    for r in reqs:
        if r["len"] < len(r["toks"]):
            segs.append(Seg(SEG_PREFILL, r["toks"][r["len"]:], r["len"], r["pages"], sample=True))
            r["len"] = len(r["toks"])
        else:
            t = int(rng.integers(0, arch.vocab))
            r["toks"].append(t)
            segs.append(Seg(SEG_DECODE, [t], r["len"], r["pages"], sample=True))
            r["len"] += 1
    eng.step(segs)
    # steps 3..: decode rows crossing page boundaries, fused with a finetuning window
    ft_toks = [int(t) for t in rng.integers(0, arch.vocab, 96)]
    ft_pages = [int(free.pop()) for _ in range(6)]
    l = 0
    for s in (40, 56):
        segs = []
        for r in reqs:
            t = int(rng.integers(0, arch.vocab))
            r["toks"].append(t)
            segs.append(Seg(SEG_DECODE, [t], r["len"], r["pages"], sample=True))
            r["len"] += 1
        segs.append(Seg(SEG_FT_FWD, ft_toks[l:l + s], l, ft_pages, adapter=True))
        tg = [ft_toks[i + 1] if i + 1 < 96 else -1 for i in range(l, l + s)]
        eng.step(segs, ft={"phase": FT_FORWARD, "seq_len": 96, "l": l, "s": s, "targets": tg})
        l += s
    for _ in range(12):
        segs = []
        for r in reqs:
            t = int(rng.integers(0, arch.vocab))
            r["toks"].append(t)
            segs.append(Seg(SEG_DECODE, [t], r["len"], r["pages"], sample=True))
            r["len"] += 1
        eng.step(segs)
    for r in reqs + [{"toks": ft_toks, "pages": ft_pages, "len": 96}]:
        k, v = eng.read_kv(0, r["pages"], r["len"])
        ek = _expected_kv(W, r["toks"][:r["len"]], "wk")
        ev = _expected_kv(W, r["toks"][:r["len"]], "wv")
        bad_k = np.argwhere(k != ek)
        bad_v = np.argwhere(v != ev)
        assert bad_k.size == 0, ("K slot mismatch (position, column)", bad_k[:5], r["pages"])
        assert bad_v.size == 0, ("V slot mismatch (position, column)", bad_v[:5], r["pages"])
    after = eng.read_kv(0, untouched, len(untouched) * P)
    assert np.array_equal(before[0], after[0]) and np.array_equal(before[1], after[1]), \
        "a page owned by no request was written"
    eng.close()


def test_kv_pages_llama_arch_within_one_ulp():
    arch = O.Arch(n_layers=2, hidden=512, n_heads=4, n_kv_heads=2, head_dim=128, ffn=512,
                  vocab=128, lora_rank=8, norm="rms", act="swiglu", rope=True, qkv_bias=True,
                  rope_theta=10000.0)
    W = O.init_general(arch, 7)
    eng = Engine(arch_config(arch, page_size=P, n_pages=64, max_tokens=256, max_ft_len=16,
                             max_segments=16))
    eng.load_weights(W)
    rng = np.random.default_rng(3)
    free = list(rng.permutation(64))
    reqs = []
    for plen in (3, 31, 70):
        toks = [int(t) for t in rng.integers(0, arch.vocab, plen)]
        reqs.append({"toks": toks, "pages": [int(free.pop()) for _ in range((plen + 8 + P - 1) // P)],
                     "cache": O.QkvCache(arch, plen + 8)})
    eng.step([Seg(SEG_PREFILL, r["toks"], 0, r["pages"], sample=True) for r in reqs])
    for r in reqs:
        O.forward_window(arch, W, r["toks"], 0, r["cache"], lora=False, emu=True)
    for _ in range(4):
        segs = []
        for r in reqs:
            t = int(rng.integers(0, arch.vocab))
            segs.append(Seg(SEG_DECODE, [t], len(r["toks"]), r["pages"], sample=True))
            O.forward_window(arch, W, [t], len(r["toks"]), r["cache"], lora=False, emu=True)
            r["toks"].append(t)
        eng.step(segs)
    for r in reqs:
        n = len(r["toks"])
        for layer in range(arch.n_layers):
            k, v = eng.read_kv(layer, r["pages"], n)
            ek, ev = r["cache"].saved[layer].k[:n], r["cache"].saved[layer].v[:n]
            for got, exp, nm in ((k, ek, "K"), (v, ev, "V")):
                # two bf16 roundings (GEMM epilogue, then RoPE of the rounded value) of numbers
                # that differ from the oracle's only in fp32-vs-f64 accumulation: a 1-ulp flip
                # at the first can carry through the rotation, so <= 2 ulps of the row's scale
                tol = np.abs(exp).max(axis=1, keepdims=True) * 2.0 ** -6
                assert np.all(np.abs(got - exp) <= tol), (nm, layer, np.abs(got - exp).max())
                # each stored row is (one of) the closest oracle row(s) to its own position's
                # (no slot permutation; equal tokens give equal layer-0 V rows, hence "one of")
                dist = ((got[:, None, :] - exp[None, :, :]) ** 2).sum(-1)
                own = dist[np.arange(n), np.arange(n)]
                assert np.all(own <= dist.min(1)), (nm, layer, np.flatnonzero(own > dist.min(1)))
    eng.close()
