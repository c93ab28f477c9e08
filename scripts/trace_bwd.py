"""SM-clock timeline of one CTA of the fused attention-backward kernel (cs_debug_trace; the
-DCS_TRACE build, python -m paper_2402_18789_b200.build --trace): 8B shape, FT forward over
L=8192, one backward window s=8192 at layer 31; traces CTA (x = argv[1] key block, kv head 0)
into gpurun_out/trace_<x>.json (summary: scripts/trace_summary.py)."""
import ctypes
import json
import os
import sys
os.environ.setdefault("CS_TRACE_LIB", "1")  # the -DCS_TRACE build (python -m paper_2402_18789_b200.build --trace)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2402_18789_b200 import _lib  # noqa: E402
from paper_2402_18789_b200.engine import Seg, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD  # noqa: E402

L = _lib.lib()
L.cs_debug_trace.restype = ctypes.c_int64
L.cs_debug_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]
buf = torch.zeros(64 * 4096, dtype=torch.int64, device="cuda:0")
eng = bench.make_engine(0, 8192)
ft_pages = list(range(0, 512))
toks = [(7 * i) % 1000 for i in range(8192)]
for l in range(0, 8192, 2048):
    eng.step([Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
             ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": 2048,
                 "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == 8192 else [])})
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 255
L.cs_debug_trace(cta, buf.data_ptr(), buf.numel())
eng.step([], ft={"phase": FT_BACKWARD, "seq_len": 8192, "l": 8192, "s": 8192, "layer": 31,
                 "pages": ft_pages})
torch.cuda.synchronize()
L.cs_debug_trace(-1, buf.data_ptr(), buf.numel())
v = buf.view(64, 4096).cpu().numpy()
evs, idxs = v.nonzero()
rec = [(int(e), int(i), int(v[e, i])) for e, i in zip(evs, idxs)]
json.dump(rec, open(os.path.join("gpurun_out", f"trace_{cta}.json"), "w"))
print(len(rec), "records")
