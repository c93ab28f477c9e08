"""Why is the last FT forward window (small s at l ~ 8K) slower than the cost model predicts?
Times a step of 64 decode rows + an FT forward window of s tokens at l = 0 vs l = 8192 - s,
with the engine's per-kind kernel profile."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_DECODE, SEG_FT_FWD, FT_FORWARD  # noqa: E402

eng = bench.make_engine(0, 8192)
P = 16
dec_pages = [list(range(i * 40, i * 40 + 40)) for i in range(64)]
ft_pages = list(range(64 * 40, 64 * 40 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]
decs = [Seg(SEG_DECODE, [i], 512, dec_pages[i], sample=True) for i in range(64)]
names = {0: "gemm", 1: "attn_bw", 2: "attn_bwd", 3: "attn_tc", 4: "allreduce"}


def win(l, s):
    eng.set_profiling(False)
    eng.set_profiling(True)
    out = eng.step(decs + [Seg(SEG_FT_FWD, toks[l:l + s], l, ft_pages, adapter=True)],
                   ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": s,
                       "targets": toks[l + 1:l + s + 1] + ([-1] if l + s == 8192 else [])})
    prof = {names[k]: round(eng.read_profile(k)["ms"], 2) for k in range(4)}
    return round(out["ms"], 2), prof


s = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for rep in range(2):
    eng.reset_ft()
    print("l=0      ", win(0, s), flush=True)
    eng.reset_ft()
    l = 0
    while l < 8192 - s:
        w = min(2048, 8192 - s - l)
        eng.step([Seg(SEG_FT_FWD, toks[l:l + w], l, ft_pages, adapter=True)],
                 ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": w, "targets": toks[l + 1:l + w + 1]})
        l += w
    print(f"l={l:5d}  ", win(l, s), flush=True)
