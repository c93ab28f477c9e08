"""Stress the finetuning backward over irregular window sizes at the 8B shape: a forward over
L=8192, then layers 31 and 30 backward in windows of mixed sizes (1 token .. 2K, odd sizes
around tile edges).  Each window is printed before it runs (cs_step synchronises), so a hang
names its window."""
import os
import random
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD  # noqa: E402

eng = bench.make_engine(0, 8192)
ft_pages = list(range(64 * 40, 64 * 40 + 512))
toks = [(7 * i) % 1000 for i in range(8192)]
for l in range(0, 8192, 2048):
    eng.step([Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
             ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": 2048,
                 "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == 8192 else [])})
sizes = [1, 2, 3, 5, 7, 8, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129, 200, 255, 256, 257,
         511, 512, 513, 1000, 1024, 1500, 2048]
rng = random.Random(int(os.environ.get("SEED", "1")))
for layer in (31, 30):
    lj = 8192
    while lj > 0:
        s = min(lj, rng.choice(sizes))
        print(f"layer {layer} l_j={lj} s={s}", flush=True)
        eng.step([], ft={"phase": FT_BACKWARD, "seq_len": 8192, "l": lj, "s": s, "layer": layer,
                         "pages": ft_pages})
        lj -= s
print("done", flush=True)
