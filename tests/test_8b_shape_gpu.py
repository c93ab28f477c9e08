"""Parity at the bench geometry: LLaMA-3.1-8B layer shapes (h=4096,
Hq 32 / Hkv 8, d=128, f=14336, r=16, RoPE theta 5e5) for 2 layers, a 4096-token finetuning
sequence in two 2048-token windows (the second at 2K-4K context) fused with 64 decode rows,
then two 2048-token backward windows per layer -- the shapes that run the CTA-pair GEMM with
its tail-wave K split, attn_fwd_tc2 over 16 KV tiles, the fused attention backward
attn_bwd_fused_kernel<4> (dQ reduce-added across 32 key blocks), the 1024-row CE head-chunk
loop and the MN-major dX GEMMs.  The vocabulary is reduced
to 16384 (the head loop and its chunking do not depend on V; the f64 oracle's [4096, V] logits
would be 4 GB at V=128256).  Checked like tests/test_coserve_gpu.py: against the bf16
rounding-point oracle at 1e-2 (or 2x its measured self-drift) and the f64 oracle under the
bf16 storage floor -- both restating tiny_model.hpp:181-327 in the LLaMA generalisation."""
import numpy as np
import pytest

from oracle import coserve_oracle as O
from paper_2402_18789_b200.engine import (Engine, Seg, arch_config, SEG_DECODE, SEG_PREFILL,
                                          SEG_FT_FWD, FT_FORWARD, FT_BACKWARD)
from tests.test_coserve_gpu import (EMU_TOL, FLOOR_DEEP, Sensitivity, _log, gate_grads,
                                    gate_loss)

pytestmark = pytest.mark.gpu

ARCH_8B2 = O.Arch(n_layers=2, hidden=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336,
                  vocab=16384, lora_rank=16, norm="rms", act="swiglu", rope=True, qkv_bias=False,
                  rope_theta=500000.0)


@pytest.mark.timeout(1800)
def test_llama8b_shape_two_layers_parity():
    arch = ARCH_8B2
    P = 16
    L, WIN = 4096, 2048
    W = O.init_general(arch, 21)
    rng = np.random.default_rng(8)
    toks = [int(t) for t in rng.integers(0, arch.vocab, L)]
    eng = Engine(arch_config(arch, page_size=P, n_pages=1024, max_tokens=WIN + 128, max_ft_len=L,
                             max_segments=80))
    eng.load_weights(W)
    free = list(range(1023, -1, -1))
    ft_pages = [free.pop() for _ in range(L // P)]
    reqs = []
    for i in range(64):
        plen = int(rng.integers(4, 12))
        reqs.append({"toks": [int(t) for t in rng.integers(0, arch.vocab, plen)],
                     "pages": [free.pop() for _ in range(2)], "check": i % 8 == 0})
    for r in reqs:
        if r["check"]:
            r["c64"], r["ce"] = O.QkvCache(arch, 32), O.QkvCache(arch, 32)
    ld, le = [], []

    def check(out, idx, r, new, pos):
        a, _ = O.forward_window(arch, W, new, pos, r["c64"], lora=False)
        b, _ = O.forward_window(arch, W, new, pos, r["ce"], lora=False, emu=True)
        ld.append(O.scaled_err(out["logits"][idx], a[-1]))
        le.append(O.scaled_err(out["logits"][idx], b[-1]))

    out = eng.step([Seg(SEG_PREFILL, r["toks"], 0, r["pages"], sample=True) for r in reqs],
                   want_logits=True)
    for i, r in enumerate(reqs):
        if r["check"]:
            check(out, i, r, r["toks"], 0)
    loss_sum = 0.0
    for l in range(0, L, WIN):
        segs = []
        for r in reqs:
            t = int(rng.integers(0, arch.vocab))
            r["new"] = t
            segs.append(Seg(SEG_DECODE, [t], len(r["toks"]), r["pages"], sample=True))
        segs.append(Seg(SEG_FT_FWD, toks[l:l + WIN], l, ft_pages, adapter=True))
        tg = [toks[i + 1] if i + 1 < L else -1 for i in range(l, l + WIN)]
        out = eng.step(segs, ft={"phase": FT_FORWARD, "seq_len": L, "l": l, "s": WIN, "targets": tg},
                       want_logits=True)
        loss_sum += out["loss_sum"]
        for i, r in enumerate(reqs):
            if r["check"]:
                check(out, i, r, [r["new"]], len(r["toks"]))
            r["toks"].append(r["new"])
    kvg, dys = {}, {}
    for n in (1, 0):
        for lj in (L, L - WIN):
            eng.step([], ft={"phase": FT_BACKWARD, "seq_len": L, "l": lj, "s": WIN, "layer": n,
                             "pages": ft_pages})
        if n == 1:
            kvg[1] = eng.kvgrad(L)
            dys[1] = eng.read_dy(L)
    _log({"test": "llama8b_shape", "q": "logits", "gpu_vs_f64": max(ld), "gpu_vs_emu": max(le)})
    assert max(ld) < 0.04, ld
    assert max(le) <= EMU_TOL, le
    O.clear_weight_cache()
    tr = O.forward_full(arch, W, toks)
    bw = O.backward_full(arch, W, tr)
    tr_loss = tr["loss"]
    del tr
    te = O.forward_full(arch, W, toks, emu=True)
    be = O.backward_full(arch, W, te)
    gate_loss("llama8b_shape", loss_sum / (L - 1), {"loss": tr_loss}, te)
    del te
    gate_grads("llama8b_shape", arch, eng, bw, be, kvg, dys, floor_deep=FLOOR_DEEP,
               sens=Sensitivity(arch, W, toks, clean=be, trials=2))
    O.clear_weight_cache()
    eng.close()
