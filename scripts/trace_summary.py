"""Summarise an attention-backward CTA trace (gpurun_out/trace_<cta>.json from trace_bwd.py):
per-tile event times and median intervals.  Events: 30 S/dP issue, 31 dV/dK/dQ issue,
40 elementwise start (warp 4), 41 its x ring wait done, 43 its P/dS buffer wait done, 42
elementwise end (warp 4), 32 S issuer's Q/dO wait done, 33 G issuer's P/dS-ready wait done,
50 dQ warps see dQ^T."""
import json
import sys

rec = json.load(open(sys.argv[1]))
t0 = min(r[2] for r in rec)
by = {}
for ev, idx, t in rec:
    by.setdefault(ev, {})[idx] = t - t0


def med(x):
    x = sorted(x)
    return x[len(x) // 2] if x else None


for i in range(0, 8):
    print(i, [f"{ev}:{by[ev][i]}" for ev in [34, 37, 35, 36, 30, 40, 41, 43, 42, 31, 38, 50, 51] if i in by.get(ev, {})])
ks = sorted(by[30])
print("tiles", len(ks), "median S issue spacing", med([by[30][k + 1] - by[30][k] for k in ks[:-1]]))
pairs = [("S issue -> E start", 30, 40, 0), ("E start -> E end", 40, 42, 0), ("E end -> dVdKdQ issue", 42, 31, 0),
         ("dVdKdQ issue -> next S issue", 31, 30, 1), ("E end -> next E start", 42, 40, 1),
         ("S issue -> next S issue", 30, 30, 1), ("E start -> x ready", 40, 41, 0),
         ("x ready -> P/dS buffer free", 41, 43, 0), ("buffer free -> E end", 43, 42, 0),
         ("prev S issue -> Q ready", 30, 32, 1), ("Q ready -> S issue", 32, 30, 0),
         ("E end -> issuer sees pds", 42, 33, 0), ("Q/dO TMA issue -> issuer sees it", 34, 32, 0), ("issuer sees pds -> dVdKdQ issue", 33, 31, 0),
         ("S issue -> next sd_full seen (E start)", 30, 40, 0), ("dVdKdQ issue -> E sees buffer free (next tile)", 31, 43, 1),
         ("dVdKdQ issue -> dQ warps see dQ", 31, 50, 0), ("dQ seen -> next dVdKdQ issue", 50, 31, 1),
         ("Q ready(seen by S issuer) -> S issue", 32, 30, 0)]
for name, a, b, off in pairs:
    print(f"{name:32s}", med([by[b][i + off] - by[a][i] for i in by.get(a, {}) if i + off in by.get(b, {})]))
