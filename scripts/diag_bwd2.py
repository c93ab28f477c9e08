"""Dump ΔKVAccum after each backward window of layer 1 (d=128 scenario) for A/B of the
attention-backward kernels: python scripts/diag_bwd2.py OUT.npz [windows...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from oracle import coserve_oracle as O  # noqa: E402
from paper_2402_18789_b200.engine import Engine, Seg, arch_config, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD  # noqa: E402
from tests.test_coserve_gpu import ARCH_D128  # noqa: E402

out = sys.argv[1]
wins = [int(x) for x in sys.argv[2:]] or [100, 200]
arch = ARCH_D128
W = O.init_general(arch, 7)
toks = list(np.random.default_rng(9).integers(0, arch.vocab, 300))
L = len(toks)
eng = Engine(arch_config(arch, page_size=16, n_pages=256, max_tokens=512, max_ft_len=L, max_segments=64))
eng.load_weights(W)
pages = list(range(20, 20 + (L + 15) // 16))
eng.step([Seg(SEG_FT_FWD, toks, 0, pages, adapter=True)],
         ft={"phase": FT_FORWARD, "seq_len": L, "l": 0, "s": L, "targets": toks[1:] + [-1]})
res = {}
lj = L
for k, s in enumerate(wins):
    eng.step([], ft={"phase": FT_BACKWARD, "seq_len": L, "l": lj, "s": s, "layer": 1, "pages": pages})
    dk, dv = eng.kvgrad(L)
    res[f"dk{k}"], res[f"dv{k}"] = dk, dv
    lj -= s
np.savez(out, **res)
print("saved", out, wins)
