"""A short 8B co-serving sequence for ncu: 4 forward-phase iterations (64 decode rows + a
2048-token finetuning window each, contexts 0..6144) then one backward-phase iteration
(64 decode rows + an 8192-token backward window at layer 31)."""
import sys
sys.path.insert(0, ".")
import bench
from paper_2402_18789_b200.engine import Seg, SEG_DECODE, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD

eng = bench.make_engine(0, 8192)
P, ctx, nd = 16, 512, 64
dec_pages = [list(range(i * 40, i * 40 + 40)) for i in range(nd)]
ft_pages = list(range(nd * 40, nd * 40 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]


def decs():
    return [Seg(SEG_DECODE, [i], ctx, dec_pages[i], sample=True) for i in range(nd)]


for l in range(0, 8192, 2048):
    out = eng.step(decs() + [Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
                   ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": 2048,
                       "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == 8192 else [])})
    print("fwd", l, round(out["ms"], 2), flush=True)
out = eng.step(decs(), ft={"phase": FT_BACKWARD, "seq_len": 8192, "l": 8192, "s": 8192,
                           "layer": 31, "pages": ft_pages})
print("bwd", round(out["ms"], 2), flush=True)
