"""tcgen05 GEMM vs cuBLAS (torch.matmul) at the 8B backward-window shapes (M = window rows):
dX of gate||up (K = 2f), dm = [dY | dU] [W_down^T ; A^T] (K = h + 64), dX of QKV / O; plus the
forward gate||up at M = 2048.  CUDA events, L2 flushed, median of 7."""
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


def t(fn):
    ts = []
    for _ in range(7):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return sorted(ts)[3]


for name, M, N, K, mn, epi in (("gate_up_dx", 8192, 4096, 28672, 1, 1), ("dm", 8192, 14336, 4160, 1, 0),
                               ("qkv_dx", 8192, 4096, 6144, 1, 1), ("o_dx(dO)", 8192, 4096, 4096, 1, 0),
                               ("gate_up_fwd", 2048, 28672, 4096, 0, 0), ("gate_up_dx_2k", 2048, 4096, 28672, 1, 1)):
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(K, N, device=dev).bfloat16() if mn else torch.randn(N, K, device=dev).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.float32 if epi == 1 else torch.bfloat16)

    def ours():
        if mn:
            rc = L.cs_gemm_bf16_mn(A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, M, N, K, epi, 0, 0, st)
        else:
            rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, epi, None, 0, 0, st)
        assert rc == 0

    Bt = B if mn else B.T
    def cub():
        torch.matmul(A, Bt)
    to, tc = t(ours), t(cub)
    fl = 2.0 * M * N * K
    print(json.dumps({"op": name, "M": M, "N": N, "K": K, "ours_ms": round(to, 4), "ours_tflops": round(fl / to / 1e9, 1),
                      "cublas_ms": round(tc, 4), "cublas_tflops": round(fl / tc / 1e9, 1)}), flush=True)
