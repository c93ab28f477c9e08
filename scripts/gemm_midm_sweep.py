"""Mid-M GEMM sweep: device time of cs_gemm_bf16 for the co-serving loop's projection shapes at
M = 256..2112 rows (8B: gate||up N=28672 K=4096, QKV N=6144 K=4096, O N=4096 K=4096 (fp32
residual add), down N=4096 K=14336 (fp32 residual add)); CUDA events, L2 flushed, median of 5.
Run once per dispatch setting (e.g. CS_GEMM_2SM=0 forces the one-CTA kernel) and compare.

    python scripts/gemm_midm_sweep.py [M,M,...] > out.jsonl
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
shapes = [("gate_up", 28672, 4096, 0), ("qkv", 6144, 4096, 0), ("o", 4096, 4096, 2), ("down", 4096, 14336, 2)]
MS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else \
    [256, 320, 384, 439, 512, 586, 640, 704, 768, 896, 1024, 1152, 1280, 1536, 1728, 2112]
for M in MS:
    for name, N, K, epi in shapes:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if epi == 0 else torch.float32)

        def run():
            rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, epi, None, 0, 0, st)
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
        t = sorted(ts)[2]
        print(json.dumps({"M": M, "shape": name, "N": N, "K": K, "epi": epi, "us": round(t * 1e3, 1),
                          "tflops": round(2.0 * M * N * K / (t * 1e-3) / 1e12, 1),
                          "env2sm": os.environ.get("CS_GEMM_2SM", "1"),
                          "bf16_split": os.environ.get("CS_GEMM_BF16_SPLIT", "1")}), flush=True)
        del A, B, C
