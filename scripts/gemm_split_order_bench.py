"""fp32-output GEMMs that take a uniform K split (LM-head dH = dlogits U with K = V; the small /
mid-M O / down projections, the LoRA products): device time (CUDA events, L2 flushed, median of
5) and max relative error vs a torch fp32 reference.

    python scripts/gemm_split_order_bench.py
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
for name, M, N, K, epi in (("lm_head_dH", 1024, 4096, 128256, 1), ("lm_head_dH_2k", 2048, 4096, 128256, 1),
                           ("down_M81", 81, 4096, 14336, 2), ("o_M128", 128, 4096, 4096, 2),
                           ("down_M640", 640, 4096, 14336, 2), ("lora_u_2k", 2048, 16, 14336, 1)):
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(N, K, device=dev).bfloat16()
    C = torch.zeros(M, N, device=dev)
    ref = A.float() @ B.float().T

    def run():
        rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, epi, None, 0, 0, st)
        assert rc == 0, L.cs_last_error()
    C.zero_()
    run()
    err = ((C - ref).abs().max() / ref.abs().max()).item()
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
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "us": round(t * 1e3, 1),
                      "tflops": round(2.0 * M * N * K / (t * 1e-3) / 1e12, 1),
                      "rel_err" if epi == 1 else "rel_err_vs_add": err}), flush=True)
    del A, B, C, ref
