"""Time the tcgen05 GEMM at the LLaMA-8B projection shapes (CUDA events, L2 flushed)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_18789_b200 import _lib  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14400)}
res = []
for T in [int(x) for x in (sys.argv[1:] or ["64", "512", "2048", "4096", "8192"])]:
    for name, (N, K) in shapes.items():
        A = torch.randn(T, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        epi = 2 if name in ("o", "down") else 0
        C = torch.zeros(T, N, device=dev, dtype=torch.float32 if epi else torch.bfloat16)
        st = torch.cuda.current_stream().cuda_stream

        def run():
            rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, T, N, K, epi,
                                None, 0, 0, st)
            assert rc == 0, L.cs_last_error()
        for _ in range(3):
            run()
        times = []
        for _ in range(10):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run()
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
        t = sorted(times)[len(times) // 2]
        tf = 2.0 * T * N * K / (t * 1e-3) / 1e12
        gbs = (T * K * 2 + N * K * 2 + T * N * (4 if epi else 2)) / (t * 1e-3) / 1e9
        # torch reference time
        Af, Bf = A, B
        for _ in range(3):
            torch.matmul(Af, Bf.T)
        ts = []
        for _ in range(10):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.matmul(Af, Bf.T)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        tt = sorted(ts)[len(ts) // 2]
        r = {"T": T, "op": name, "ms": round(t, 4), "tflops": round(tf, 1), "gbs": round(gbs, 1),
             "cublas_ms": round(tt, 4), "cublas_tflops": round(2.0 * T * N * K / (tt * 1e-3) / 1e12, 1)}
        print(json.dumps(r), flush=True)
        res.append(r)
