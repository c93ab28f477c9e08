"""The bench's co-serving loop for a profiler: offline profile first (outside the NVTX range),
then `--iters` iterations of the 8B co-serving loop at `--rate` req/s inside the NVTX range
"coserve", with the clock advanced by the planner's predicted latency (sim_clock) so the plan
sequence does not depend on the profiler's slowdown.

  ncu --nvtx --nvtx-include "coserve/" --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python scripts/ncu_coserve.py
  python scripts/ncu_coserve.py --reduce gpurun_out/launches.csv   # per-kernel shares
"""
import argparse
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def reduce(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            t[name] += float(r[vi].replace(",", ""))
            n[name] += 1
    tot = sum(t.values())
    print(f"{'kernel':44s} {'launches':>8s} {'share':>7s} {'avg us':>9s}")
    for k, v in sorted(t.items(), key=lambda kv: -kv[1]):
        print(f"{k[:44]:44s} {n[k]:8d} {100 * v / tot:6.2f}% {v / n[k] / 1000:9.1f}")
    print(f"total {tot / 1e6:.2f} ms over {sum(n.values())} launches")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, default=20.0)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--reduce", default="")
    ap.add_argument("--fixed-profile", action="store_true",
                    help="skip the offline profile (a recorded B200 profile instead): only the "
                         "loop's own launches run, e.g. for CS_GEMM_LOG shape censuses")
    a = ap.parse_args()
    if a.reduce:
        return reduce(a.reduce)
    import torch
    import bench
    from paper_2402_18789_b200.engine import coserve_run
    eng = bench.make_engine(0, 8192)
    if a.fixed_profile:  # bench.py's offline profile on a B200 (profiles/r1_bench_latest.log)
        prof = {"t0_ms": 5.46, "decode_ms_per_row": 0.0105, "prefill_ms_per_token": 0.0178,
                "slope_ms_per_token": 0.01864, "bwd_token_weight": 0.02548,
                "attn_fwd_ms_per_token_ctx": 7.99e-07, "attn_bwd_ms_per_token_ctx": 8.65e-08,
                "bwd_layer0_weight": 0.2545}
    else:
        prof = bench.offline_profile(eng, 8192)
    c = bench.coserve_config(a.rate, prof, a.iters, 0, 8192, seed=7)
    c.sim_clock, c.adaptive = 1, 0
    torch.cuda.nvtx.range_push("coserve")
    st, log = coserve_run(eng, c)
    torch.cuda.nvtx.range_pop()
    print({k: st[k] for k in ("ft_fwd_tokens", "ft_bwd_tokens", "gpu_launches", "timed_ms", "timed_device_ms")})


if __name__ == "__main__":
    main()
