"""Probe (bn, splits) overrides of cs_gemm_bf16 for given shapes against the dispatcher's choice
(bn = splits = 0); fp32 residual-add epilogue; CUDA events, L2 flushed, median of 5.

    python scripts/gemm_cfg_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_18789_b200 import _lib  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
for (M, N, K, epi) in ((576, 4096, 14400, 2), (1088, 4096, 14400, 2), (2880, 4096, 4096, 2), (576, 4096, 4096, 2)):
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(N, K, device=dev).bfloat16()
    C = torch.zeros(M, N, device=dev)
    out = []
    for bn, sp in [(0, 0)] + [(b, s) for b in (128, 256) for s in (1, 2, 3, 4, 5, 6, 8)]:
        def run():
            rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, epi, None, bn, sp, st)
            assert rc == 0, L.cs_last_error()
        run()
        ts = []
        for _ in range(5):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        out.append((bn, sp, round(sorted(ts)[2] * 1e3, 1)))
    best = min(out[1:], key=lambda x: x[2])
    print(json.dumps({"M": M, "N": N, "K": K, "epi": epi, "default_us": out[0][2], "best": best,
                      "all": out}), flush=True)
    del A, B, C
