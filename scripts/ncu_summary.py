"""Summarise an ncu --set full report (.ncu-rep) into the per-launch numbers the roofline
claims rest on: duration, tensor-pipe activity, DRAM bytes and throughput, L2 hit rate, SM
throughput, registers.  python scripts/ncu_summary.py REPORT.ncu-rep [> profiles/...txt]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_active_%"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc_inst_%"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        print(f"kernel: {r[h.index('Kernel Name')]}")
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {name:24s} {r[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
