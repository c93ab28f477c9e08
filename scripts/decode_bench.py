"""One decode-only step on 8B-shaped layers (B rows at context c) -- the target for
`ncu --set full -k regex:attn_decode` (scripts/kernel_sweep.py covers the sweep)."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.kernel_sweep import make, P  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_DECODE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--ctx", type=int, default=2048)
ap.add_argument("--layers", type=int, default=1)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
per = (a.ctx + P) // P + 1
eng = make(a.layers, a.B * per + 16, 256)
segs = [Seg(SEG_DECODE, [i % 1000], a.ctx, list(range(i * per, (i + 1) * per))) for i in range(a.B)]
for _ in range(a.steps):
    print(eng.step(segs)["ms"])
