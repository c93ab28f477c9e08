"""Print the headline ncu metrics (duration, tensor pipe, shared-memory wavefronts, DRAM, L2) and
the top stall / shared-wavefront source lines of one kernel in an .ncu-rep."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k in want:
    if k in h:
        print(f"{k:90s} {v[h.index(k)]}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    data = rows[2:]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(f(r[ix["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
    print("\ntop stall lines (% of samples) and their dominant stall reason")
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    for r in sorted(data, key=lambda r: -f(r[ix["Warp Stall Sampling (All Samples)"]]))[:int(sys.argv[2])]:
        rs = max(reasons, key=lambda k: f(r[ix[k]]))
        print(f"{f(r[ix['Warp Stall Sampling (All Samples)']]) / tot * 100:5.1f}  {r[ix['Address']][-5:]}  {rs:18s} {r[ix['Source']][:90]}")
