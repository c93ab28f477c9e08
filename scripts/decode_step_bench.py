"""Decode-only co-serving step (8B shape, all 32 layers): `--rows` decode rows at 300-500-token
contexts, device time per step (engine CUDA events, median of `--reps`) -- the iterations whose
projections are weight streams (M = rows)."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_DECODE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=81)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
eng = bench.make_engine(0, 8192)
segs = [Seg(SEG_DECODE, [i % 1000], 300 + i, list(range(40 * i, 40 * i + 40)), sample=True) for i in range(a.rows)]
ts = []
for r in range(a.reps + 5):
    out = eng.step(segs)
    if r >= 5:
        ts.append(out["ms"])
print(f"rows={a.rows} step {statistics.median(ts):.3f} ms (min {min(ts):.3f})", flush=True)
