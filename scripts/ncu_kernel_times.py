"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel and grid shape.

usage: python scripts/ncu_kernel_times.py launches.csv
"""
import collections
import csv
import statistics
import sys


def main(path):
    lines = open(path).read().splitlines()
    start = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    by = collections.defaultdict(list)
    for r in csv.DictReader(lines[start:]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        by[(r["Kernel Name"][:60], r["Grid Size"])].append(float(r["Metric Value"]) * scale)
    for (k, g), v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:60s} grid {g:14s} n={len(v):5d} mean {statistics.mean(v):8.2f} us  "
              f"median {statistics.median(v):8.2f} us  total {sum(v) / 1e3:8.2f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
