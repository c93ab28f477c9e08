"""DRAM traffic of the tcgen05 GEMM vs its algorithmic bytes, for bench.py's `roofline.traffic`.

Run under ncu (one GPU):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_tn --csv \
      --log-file gpurun_out/gemm_traffic.csv python scripts/gemm_traffic.py
then `python scripts/gemm_traffic.py --reduce gpurun_out/gemm_traffic.csv` writes
profiles/gemm_traffic.json: DRAM bytes per launch (ncu) next to the engine's algorithmic
bytes per launch (2*(M*K + N*K) + M*N*out_bytes, summed by its live profiler) over the same
sequence (scripts/ncu_step.py's co-serving iterations: 64 decode rows + 2048-token FT windows,
then an 8192-token backward window).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import bench
    from paper_2402_18789_b200.engine import Seg, SEG_DECODE, SEG_FT_FWD, FT_FORWARD, FT_BACKWARD
    eng = bench.make_engine(0, 8192)
    nd, ctx = 64, 512
    dec_pages = [list(range(i * 40, i * 40 + 40)) for i in range(nd)]
    ft_pages = list(range(nd * 40, nd * 40 + 512))
    toks = [(7 * i) % 1000 for i in range(8192)]
    decs = [Seg(SEG_DECODE, [i], ctx, dec_pages[i], sample=True) for i in range(nd)]
    eng.set_profiling(True)
    for l in range(0, 8192, 2048):
        eng.step(decs + [Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
                 ft={"phase": FT_FORWARD, "seq_len": 8192, "l": l, "s": 2048,
                     "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == 8192 else [])})
    eng.step(decs, ft={"phase": FT_BACKWARD, "seq_len": 8192, "l": 8192, "s": 8192, "layer": 31,
                       "pages": ft_pages})
    g = eng.read_profile(0)
    out = {"algorithmic_bytes": g["bytes"], "flops": g["flops"], "launches": g["launches"]}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "gemm_traffic_alg.json"), "w"))
    print(json.dumps(out))


def reduce(path):
    rows = list(csv.reader(open(path)))
    hdr, tot, ids = None, 0.0, set()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v = float(d["Metric Value"])
                unit = d.get("Metric Unit", "byte")
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                tot += v
                ids.add(d["ID"])
    alg = json.load(open(os.path.join(ROOT, "gpurun_out", "gemm_traffic_alg.json")))
    n = len(ids)
    res = {"dram_bytes_per_launch": tot / n, "algorithmic_bytes_per_launch": alg["algorithmic_bytes"] / alg["launches"],
           "launches_ncu": n, "launches_engine": alg["launches"],
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:gemm_tn "
                     "over scripts/gemm_traffic.py (cold-cache, serialised replays)"}
    res["traffic_over_algorithmic"] = res["dram_bytes_per_launch"] / res["algorithmic_bytes_per_launch"]
    json.dump(res, open(os.path.join(ROOT, "profiles", "gemm_traffic.json"), "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--reduce":
        reduce(sys.argv[2])
    else:
        run()
