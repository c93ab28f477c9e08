"""A/B the attention forward paths on the 8B shape: 2048-token FT windows at l=0..6144 with 64
decode rows on the two-query-tile tcgen05 kernel, device
time of the attention kernels from the engine's CUDA events."""
import os
import sys
sys.path.insert(0, ".")
import bench
from paper_2402_18789_b200.engine import Seg, SEG_DECODE, SEG_FT_FWD, FT_FORWARD

eng = bench.make_engine(0, 8192)
nd = 64
dec_pages = [list(range(i * 40, i * 40 + 40)) for i in range(nd)]
ft_pages = list(range(nd * 40, nd * 40 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]
eng.set_profiling(True)
for l in range(0, 8192, 2048):
    out = eng.step([Seg(SEG_DECODE, [i], 512, dec_pages[i], sample=True) for i in range(nd)] +
                   [Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
                   ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": 2048,
                       "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == 8192 else [])})
    a = eng.read_profile(3)
    d = eng.read_profile(1)
    g = eng.read_profile(0)
    print(f"l={l} step {out['ms']:.2f} ms  "
          f"attn(tc) {a['ms']:.2f} ms {a['flops']/max(a['ms'],1e-9)/1e9:.0f} TFLOP/s  decode {d['ms']:.2f} ms  "
          f"gemm {g['ms']:.2f} ms {g['flops']/g['ms']/1e9:.0f} TFLOP/s", flush=True)
    eng.set_profiling(False); eng.set_profiling(True)
