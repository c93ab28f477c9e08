"""Attention forward (tcgen05 kernel, engine profile kind 3) at the bench's forward-iteration
compositions: one FT window of s tokens at context l, optionally next to a 512-token prefill
chunk (context 0) and 80 decode rows -- TFLOP/s per call shape (8B, one layer's call; median of
`--reps` steps).

    python scripts/attn_mix_bench.py [--reps 5]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_DECODE, SEG_PREFILL, SEG_FT_FWD, FT_FORWARD  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
eng = bench.make_engine(0, 8192)
nd = 80
dec_pages = [list(range(i * 40, i * 40 + 40)) for i in range(nd)]
pre_pages = list(range(nd * 40, nd * 40 + 40))
ft_pages = list(range(nd * 40 + 64, nd * 40 + 64 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]
for s in (512, 1024, 2048):
    for l in (0, 2048, 4096, 7168 - s + 1024 if s < 2048 else 6144):
        for mix in (0, 1):
            segs = []
            if mix:
                segs += [Seg(SEG_DECODE, [i], 400, dec_pages[i], sample=True) for i in range(nd)]
                segs += [Seg(SEG_PREFILL, toks[:512], 0, pre_pages, sample=True)]
            segs += [Seg(SEG_FT_FWD, toks[l:l + s], l, ft_pages, adapter=True)]
            res = []
            for rep in range(a.reps + 1):
                eng.reset_ft()
                for x in range(0, l, 2048):  # the FT cache must hold positions [0, l)
                    w = min(2048, l - x)
                    eng.step([Seg(SEG_FT_FWD, toks[x:x + w], x, ft_pages, adapter=True)],
                             ft={"phase": FT_FORWARD, "seq_len": 8192, "l": x, "s": w,
                                 "targets": toks[x + 1:x + w + 1]})
                eng.set_profiling(True)
                eng.step(segs, ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": s,
                                   "targets": toks[l + 1:l + s + 1]})
                r = eng.read_profile(3)
                eng.set_profiling(False)
                if rep:
                    res.append((r["ms"] / max(1, r["launches"]), r["flops"] / max(1, r["launches"])))
            ms = statistics.median(x[0] for x in res)
            fl = res[0][1]
            print(f"s={s:5d} l={l:5d} {'+prefill512+80dec' if mix else 'FT window only   '}: "
                  f"{1e3 * ms:7.1f} us per call  {fl / ms / 1e9:6.0f} TFLOP/s  ({fl:.3g} FLOP)", flush=True)
