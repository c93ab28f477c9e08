"""Tile / split-K sweep of the tcgen05 GEMM at the co-serving loop's mid-M shapes (the census in
scripts/gemm_census.py): heuristic choice vs forced 1-CTA tile widths x K splits (CUDA events,
L2 flushed).  Used to fit gemm.cu's shape heuristic.

  python scripts/gemm_cfg_sweep.py [--out gpurun_out/gemm_cfg_sweep.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [  # (M, N, K, epi): 8B projections at the backward-phase iterations' inference rows
    (576, 28672, 4096, 0), (640, 28672, 4096, 0), (704, 28672, 4096, 0), (960, 28672, 4096, 0),
    (640, 4096, 14400, 2), (704, 4096, 14400, 2), (1728, 4096, 14400, 2), (2112, 4096, 14400, 2),
    (640, 6144, 4096, 0), (1728, 6144, 4096, 0), (2112, 6144, 4096, 0),
    (640, 4096, 4096, 2), (2112, 4096, 4096, 2), (1024, 4096, 128256, 1),
    (1600, 6144, 4096, 0), (1856, 6144, 4096, 0), (1984, 6144, 4096, 0), (1728, 4096, 4096, 2),
    (1600, 28672, 4096, 0), (1600, 4096, 14400, 2),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/gemm_cfg_sweep.json")
    a = ap.parse_args()
    import torch
    from paper_2402_18789_b200 import _lib
    L = _lib.lib()
    dev = torch.device("cuda:0")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    res = []
    for M, N, K, epi in SHAPES:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if epi == 0 else torch.float32)

        def timed(bn, splits):
            def run():
                rc = L.cs_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, epi,
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
            return sorted(ts)[2] * 1e3
        row = {"M": M, "N": N, "K": K, "epi": epi, "auto_us": round(timed(0, 0), 1), "forced": {}}
        for bn in (64, 128, 256):
            for sp in ((1, 2, 3, 4) if epi != 0 else (1,)):
                row["forced"][f"bn{bn}_s{sp}"] = round(timed(bn, sp), 1)
        best = min(row["forced"].items(), key=lambda kv: kv[1])
        row["best"] = best
        row["auto_tflops"] = round(2.0 * M * N * K / (row["auto_us"] * 1e-6) / 1e12, 1)
        row["best_tflops"] = round(2.0 * M * N * K / (best[1] * 1e-6) / 1e12, 1)
        res.append(row)
        print(json.dumps({k: v for k, v in row.items() if k != "forced"}), flush=True)
        del A, B, C
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
