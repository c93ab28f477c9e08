"""Host enqueue time vs device time of representative 8B co-serving steps (is any part of a
step launch-bound?).  step_async = plan checks + meta upload + every kernel launch, no sync."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_DECODE, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD  # noqa: E402

P = 16
eng = bench.make_engine(0, 8192)
dec_pages = [list(range(i * 40, i * 40 + 40)) for i in range(128)]
ft_pages = list(range(128 * 40, 128 * 40 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]


def decs(n=100):
    return [Seg(SEG_DECODE, [i], 400 + i, dec_pages[i], sample=True) for i in range(n)]


def run(segs, ft, reps=1):
    res = []
    tp = time.perf_counter()
    eng._plan(segs, ft)  # Python-side plan marshalling alone (not part of the C++ loop's cost)
    tp = (time.perf_counter() - tp) * 1e3
    print(f"  python plan marshalling {tp:.2f} ms", end="; ")
    for _ in range(reps):
        t0 = time.perf_counter()
        eng.step_async(segs, ft)
        t1 = time.perf_counter()
        dev = eng.sync()
        t2 = time.perf_counter()
        res.append(((t1 - t0) * 1e3, dev, (t2 - t0) * 1e3))
    return min(res, key=lambda r: r[2])


for l, s in ((0, 1536), (1536, 1536), (3072, 1536), (4608, 1536), (6144, 2048)):
    r = run(decs() + [Seg(SEG_FT_FWD, toks[l:l + s], l, ft_pages, adapter=True)],
            {"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": s,
             "targets": toks[l + 1:l + s + 1] + ([-1] if l + s == 8192 else [])})
    print(f"fwd l={l} s={s}: enqueue {r[0]:.2f} ms, device {r[1]:.2f} ms, wall {r[2]:.2f} ms", flush=True)
for n in range(31, 25, -1):
    r = run(decs(), {"phase": FT_BACKWARD, "seq_len": 8192, "l": 8192, "s": 8192, "layer": n,
                     "pages": ft_pages}, reps=1)
    print(f"bwd layer {n}: enqueue {r[0]:.2f} ms, device {r[1]:.2f} ms, wall {r[2]:.2f} ms", flush=True)
r = run(decs(), None)
print(f"decode only: enqueue {r[0]:.2f} ms, device {r[1]:.2f} ms, wall {r[2]:.2f} ms", flush=True)
