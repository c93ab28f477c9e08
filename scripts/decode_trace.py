"""Per-warp timeline of one decode-attention launch at the bench's operating point (experiment
build: python scripts/build_variant.py dectrace attn_decode.cu -DCS_DEC_TRACE, then
CS_LIB_PATH=paper_2402_18789_b200/variants/dectrace.so python scripts/decode_trace.py [--B 60]).
Prints the launch span, the spread of warp start times, the first-tile latency, and when the
warps finish (quantiles, us from the first warp's start), and the per-SM tile counts."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from scripts.decode_op import contexts  # noqa: E402
from scripts.kernel_sweep import make, P  # noqa: E402
from paper_2402_18789_b200 import _lib  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_DECODE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=60)
a = ap.parse_args()
L = _lib.lib()
L.cs_debug_dec_trace.argtypes = [ctypes.c_void_p]
ctxs = contexts(a.B)
pages = sum((c + P) // P + 1 for c in ctxs) + 16
eng = make(1, pages, 256)
segs, base = [], 0
for i, c in enumerate(ctxs):
    per = (c + P) // P + 1
    segs.append(Seg(SEG_DECODE, [i % 1000], c, list(range(base, base + per)), sample=True))
    base += per
for _ in range(5):
    eng.step(segs)
buf = torch.zeros(4096 * 5, dtype=torch.int64, device="cuda:0")
L.cs_debug_dec_trace(buf.data_ptr())
eng.step(segs)
torch.cuda.synchronize()
L.cs_debug_dec_trace(None)
v = buf.view(-1, 5).cpu().numpy()
v = v[v[:, 0] != 0]
t0 = v[:, 0].min()
st, first, end, tiles, sm = (v[:, 0] - t0) / 1e3, (v[:, 1] - t0) / 1e3, (v[:, 2] - t0) / 1e3, v[:, 3], v[:, 4]
q = lambda x: [round(float(np.quantile(x, p)), 2) for p in (0, 0.1, 0.5, 0.9, 1.0)]  # noqa: E731
per_sm = np.bincount(sm.astype(int), weights=tiles, minlength=148)
out = {"B": a.B, "warps": int(len(v)), "span_us": round(float(end.max()), 2),
       "start_q": q(st), "first_tile_latency_q": q(first - st), "end_q": q(end),
       "tiles_per_warp_q": q(tiles), "tiles_per_sm_mean_max": [round(float(per_sm.mean()), 1), int(per_sm.max())],
       "bytes_MB": round(float(tiles.sum()) * 16384 / 1e6, 1)}
# consumed-bytes timeline: each warp's tiles spread evenly over [first tile, end]
bins = np.zeros(int(end.max()) + 2)
for f, e, n in zip(first, end, tiles):
    if n <= 0:
        continue
    lo, hi = f, max(e, f + 1e-3)
    for b in range(int(lo), int(hi) + 1):
        ov = max(0.0, min(hi, b + 1) - max(lo, b))
        bins[b] += n * 16384 * ov / (hi - lo)
out["GBps_per_us_bin"] = [round(x / 1e3, 0) for x in bins]  # bytes per us -> GB/s
print(json.dumps(out))
