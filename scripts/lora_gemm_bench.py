"""The LoRA products of the 8B layer on the tensor cores: u = m A (M rows, N = r = 16,
K = f = 14336) and dlu = dY B^T (M rows, N = 16, K = h = 4096), fp32 out; CUDA events, L2
flushed, median of 7."""
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
for name, K in (("u=mA", 14336), ("dlu=dYB^T", 4096)):
    for M in (512, 1024, 2048, 4096, 8192):
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(16, K, device=dev).bfloat16()
        C = torch.zeros(M, 16, device=dev)
        ref = A.float() @ B.float().T

        def run():
            rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), 16, M, 16, K, 1, None, 0, 0, st)
            assert rc == 0, L.cs_last_error()
        run()
        err = ((C - ref).abs().max() / ref.abs().max()).item()
        ts = []
        for _ in range(7):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        t = sorted(ts)[3]
        print(json.dumps({"gemm": name, "M": M, "K": K, "us": round(t * 1e3, 1),
                          "GBps": round(M * K * 2 / (t * 1e-3) / 1e9, 1), "rel_err": err}), flush=True)
