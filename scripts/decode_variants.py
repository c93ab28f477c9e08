"""Decode attention A/B (CS_DEC_CFG variants): device time of the decode launches (engine CUDA
events, kind 1) on decode-only 8B-shaped steps at bench-like sizes.

  CS_DEC_CFG=23 python scripts/decode_variants.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from scripts.kernel_sweep import make, timed, P  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_DECODE  # noqa: E402

CASES = [(64, 512), (64, 1024), (32, 1024), (128, 512), (32, 4096), (8, 8192), (48, "mix")]
hbm = bench.load_peaks()[0]["hbm_gbs"]
eng = make(2, 16384 + 64, 256)
out = []
for B, c in CASES:
    if c == "mix":  # bench-like: lognormal contexts
        ctxs = [int(x) for x in np.clip(np.random.default_rng(0).lognormal(5.9, 0.8, B), 16, 4000)]
    else:
        ctxs = [c] * B
    segs, base = [], 0
    for i, cx in enumerate(ctxs):
        per = (cx + P) // P + 1
        segs.append(Seg(SEG_DECODE, [i % 1000], cx, list(range(base, base + per))))
        base += per
    ms, prof = timed(eng, lambda: eng.step(segs)["ms"], reps=10)
    a = prof[1]
    us = 1000.0 * a["ms"] / max(1, a["launches"])
    by = a["bytes"] / max(1, a["launches"])
    out.append({"B": B, "ctx": c, "us_per_launch": round(us, 2), "MB": round(by / 1e6, 2),
                "gbs": round(by / us / 1e3, 1), "hbm_frac": round(by / us / 1e3 / hbm, 4)})
    print(json.dumps(out[-1]), flush=True)
print(json.dumps({"cfg": os.environ.get("CS_DEC_CFG", "default"), "rows": out}))
