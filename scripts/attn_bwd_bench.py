"""Attention backward at the 8B shape: finetuning forward over L=8192 (4 windows of 2048), then
backward windows at layer 31 of size s ending at l_j (2048 x 4) and one 8192 window at layer 30;
`--reps` passes (engine FT state reset between them), reporting the median attention-backward
device time per window (Delta + the backward kernel(s); CUDA events of the engine profiler).

    python scripts/attn_bwd_bench.py [--reps 3]
"""
import argparse
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--window", type=int, default=0, help="layer 31 windows of this size over the whole sequence instead")
args = ap.parse_args()
a_w = args.window
eng = bench.make_engine(0, 8192)
ft_pages = list(range(64 * 40, 64 * 40 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]
res = {}
for rep in range(args.reps + 1):  # pass 0 is warm-up
    eng.reset_ft()
    for l in range(0, 8192, 2048):
        eng.step([Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
                 ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": 2048,
                     "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == 8192 else [])})
    plan = [(31, [a_w] * (8192 // a_w))] if a_w else [(31, [2048, 2048, 2048, 2048]), (30, [8192])]
    for layer, windows in plan:
        lj = 8192
        for s in windows:
            eng.set_profiling(True)
            out = eng.step([], ft={"phase": FT_BACKWARD, "seq_len": 8192, "l": lj, "s": s,
                                   "layer": layer, "pages": ft_pages})
            b = eng.read_profile(2)
            eng.set_profiling(False)
            if rep > 0:
                res.setdefault((layer, lj, s), []).append((b["ms"], b["flops"], out["ms"]))
            lj -= s
    # the remaining layers' backward windows are not needed: the next pass resets the FT state
tag = "fused"
for (layer, lj, s), v in res.items():
    ms = statistics.median(x[0] for x in v)
    fl = v[0][1]
    print(f"[{tag}] layer {layer} l_j={lj} s={s}: attn bwd {ms:.3f} ms = {fl / ms / 1e9:.0f} TFLOP/s "
          f"(min {min(x[0] for x in v):.3f}, max {max(x[0] for x in v):.3f}; step {statistics.median(x[2] for x in v):.2f} ms)",
          flush=True)
