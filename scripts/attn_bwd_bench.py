"""A/B of the attention backward at the 8B shape: finetuning forward over L=8192 (4 windows),
then backward windows at layer 31 of size s ending at l_j; reports the attention-backward
kernels' device time (CS_ATTN_TC=1 tcgen05 vs 0 mma.sync)."""
import os
import sys
sys.path.insert(0, ".")
import bench
from paper_2402_18789_b200.engine import Seg, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD

eng = bench.make_engine(0, 8192)
ft_pages = list(range(64 * 40, 64 * 40 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]
for l in range(0, 8192, 2048):
    eng.step([Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
             ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": 2048,
                 "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == 8192 else [])})
tag = os.environ.get("CS_ATTN_TC", "1")
for layer, windows in [(31, [2048, 2048, 2048, 2048]), (30, [8192])]:
    lj = 8192
    for s in windows:
        eng.set_profiling(True)
        out = eng.step([], ft={"phase": FT_BACKWARD, "seq_len": 8192, "l": lj, "s": s,
                               "layer": layer, "pages": ft_pages})
        b = eng.read_profile(2)
        g = eng.read_profile(0)
        print(f"CS_ATTN_TC={tag} layer {layer} l_j={lj} s={s}: step {out['ms']:.2f} ms, attn bwd "
              f"{b['ms']:.2f} ms = {b['flops'] / b['ms'] / 1e9:.0f} TFLOP/s, gemm {g['ms']:.2f} ms", flush=True)
        eng.set_profiling(False)
        lj -= s
