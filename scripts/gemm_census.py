"""GEMM shape census of the co-serving loop: which (M, N, K, epilogue) shapes the bench's
iterations issue, how often, and how fast each runs alone (CUDA events, L2 flushed).

  CS_GEMM_LOG=gpurun_out/gemm.log python scripts/ncu_coserve.py --iters 40
  python scripts/gemm_census.py gpurun_out/gemm.log [--top 25]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("log")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--out", default="gpurun_out/gemm_census.json")
    a = ap.parse_args()
    cnt = collections.Counter()
    for line in open(a.log):
        p = line.split()
        if len(p) == 4:
            cnt[tuple(int(x) for x in p)] += 1
    # bucket M to 64 rows (the loop's T varies every iteration) -> time representative shapes
    buck = collections.Counter()
    for (M, N, K, epi), c in cnt.items():
        buck[((M + 63) // 64 * 64, N, K, epi)] += c
    import torch
    from paper_2402_18789_b200 import _lib
    L = _lib.lib()
    dev = torch.device("cuda:0")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    # the heaviest buckets by count x flops
    order = sorted(buck.items(), key=lambda kv: -kv[1] * kv[0][0] * kv[0][1] * kv[0][2])
    for (M, N, K, epi0), c in order[:a.top]:
        # the fused epilogues (5 SwiGLU, 6 QKV RoPE + KV append) are timed as the plain bf16 one
        epi = 0 if epi0 in (5, 6) else epi0
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if epi == 0 else torch.float32)

        def run():
            rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, epi,
                                None, 0, 0, st)
            assert rc == 0, L.cs_last_error()
        for _ in range(2):
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
        t = sorted(ts)[len(ts) // 2]
        tc = []
        for _ in range(5):  # cuBLAS (torch.matmul, bf16 out) on the same operands
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch.matmul(A, B.T)
            e.record()
            torch.cuda.synchronize()
            tc.append(s.elapsed_time(e))
        tcu = sorted(tc)[len(tc) // 2]
        tf = 2.0 * M * N * K / (t * 1e-3) / 1e12
        rows.append({"M": M, "N": N, "K": K, "epi": epi0, "count": c, "us": round(t * 1e3, 1),
                     "tflops": round(tf, 1), "cublas_us": round(tcu * 1e3, 1), "total_ms": round(c * t, 2)})
        del A, B, C
    tot = sum(r["total_ms"] for r in rows)
    rows.sort(key=lambda r: -r["total_ms"])
    print(f"{'M':>6} {'N':>7} {'K':>7} {'epi':>3} {'count':>6} {'us':>8} {'TF/s':>7} {'cuBLAS us':>9} {'share':>6}")
    for r in rows:
        print(f"{r['M']:6d} {r['N']:7d} {r['K']:7d} {r['epi']:3d} {r['count']:6d} {r['us']:8.1f} "
              f"{r['tflops']:7.1f} {r['cublas_us']:9.1f} {100 * r['total_ms'] / tot:5.1f}%")
    json.dump({"unique_shapes": len(cnt), "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
