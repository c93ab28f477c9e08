"""Small-M GEMM exploration: time cs_gemm_bf16 at M in {64, 128, 256} for the 8B projection
shapes over tile widths / split-K (fp32 output), L2 flushed between runs."""
import json
import sys
import torch
sys.path.insert(0, ".")
from paper_2402_18789_b200 import _lib  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14400)}
for T in (64, 128, 256):
    for name, (N, K) in shapes.items():
        A = torch.randn(T, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.zeros(T, N, device=dev, dtype=torch.float32)
        st = torch.cuda.current_stream().cuda_stream
        best = None
        for bn in (16, 32, 64, 128, 256):
            for splits in (1, 2, 3, 4, 6, 8):
                def run():
                    rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, T, N, K, 1,
                                        None, bn, splits, st)
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
                gbs = (N * K * 2) / (t * 1e-3) / 1e9
                if best is None or t < best[0]:
                    best = (t, bn, splits, gbs)
        print(json.dumps({"T": T, "op": name, "best_ms": round(best[0], 4), "bn": best[1],
                          "splits": best[2], "weight_gbs": round(best[3], 1)}), flush=True)
