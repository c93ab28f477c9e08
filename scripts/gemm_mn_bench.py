"""K-major vs MN-major B operand at the backward dX GEMM shapes (8B): dX = dY . W^T read from
the reference-layout copy [N, K] (K-major) or from the forward copy [K, N] (MN-major)."""
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
res = []
for M in (2048, 8192, 640):
    for name, N, K, epi in (("gate_up_dx", 4096, 28672, 1), ("qkv_dx", 4096, 6144, 1),
                            ("o_dx", 4096, 4096, 0), ("head_dx", 4096, 128256, 1)):
        if name == "head_dx" and M != 2048:
            continue
        A = torch.randn(M, K, device=dev).bfloat16()
        Bnk = torch.randn(N, K, device=dev).bfloat16()
        Bkn = Bnk.T.contiguous()
        C = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if epi == 0 else torch.float32)
        out = {}
        for mode in ("k", "mn"):
            def run():
                if mode == "k":
                    rc = L.cs_gemm_bf16(A.data_ptr(), K, Bnk.data_ptr(), K, C.data_ptr(), N, M, N, K,
                                        epi, None, 0, 0, st)
                else:
                    rc = L.cs_gemm_bf16_mn(A.data_ptr(), K, Bkn.data_ptr(), N, C.data_ptr(), N, M, N,
                                           K, epi, 0, 0, st)
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
            out[mode] = {"us": round(t * 1e3, 1), "tflops": round(2.0 * M * N * K / (t * 1e-3) / 1e12, 1)}
        r = {"shape": name, "M": M, "N": N, "K": K, **out}
        res.append(r)
        print(json.dumps(r), flush=True)
        del A, Bnk, Bkn, C
json.dump(res, open("gpurun_out/gemm_mn_bench.json", "w"), indent=1)
