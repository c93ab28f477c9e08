"""Time single GEMM shapes through the C ABI (CUDA events, 50 launches after 10 warm-up, a
256 MB L2 flush between launches excluded from the timing).  A/B a launcher knob by running
it twice with the environment variable toggled, e.g. CS_GEMM_TAIL=0 / 1.

  python scripts/gemm_shape_time.py 1728x4096x14400x2 1984x4096x14400x2
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_18789_b200 import _lib  # noqa: E402


def main(shapes):
    L = _lib.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for spec in shapes:
        M, N, K, epi = (int(x) for x in spec.split("x"))
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = torch.randn(N, K, device="cuda").bfloat16()
        C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 0 else torch.float32)
        st = torch.cuda.current_stream()
        ts = []
        for i in range(60):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, epi,
                                      None, 0, 0, st.cuda_stream), "cs_gemm_bf16")
            e1.record(st)
            if i >= 10:
                ts.append((e0, e1))
        torch.cuda.synchronize()
        us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
        med = us[len(us) // 2]
        print(f"{spec:22s} median {med:8.1f} us  min {us[0]:8.1f}  {2 * M * N * K / med / 1e6:7.1f} TF/s")


if __name__ == "__main__":
    main(sys.argv[1:])
