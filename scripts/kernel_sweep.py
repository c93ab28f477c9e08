"""BASELINE config 5: kernel sweep on the LLaMA-3.1-8B layer shapes (1 B200).

  python scripts/kernel_sweep.py [--layers 4] [--out gpurun_out/kernel_sweep.json]

* decode-only: B decode rows x context c (B*c <= the KV pool, no page aliasing so every
  K/V byte comes from HBM); decode attention kernel time from the engine's CUDA events,
  algorithmic bytes = sum 2*c*kv_dim*2 B (+q/o) per layer -> GB/s and fraction of the
  measured HBM peak (MEASURED_PEAKS.json).
* finetune-only: one FT forward window s at offset l (tcgen05 attention + GEMMs), and the
  matching backward window at one layer -> TFLOP/s against the measured bf16 peak.
* mixed: T = 2048 tokens per step split between inference (64 decode rows at ctx 1024 +
  512-token prefill chunks) and an FT forward window, FT fraction 0..100 %.
The engine runs `--layers` 8B-shaped layers (per-layer kernels are identical to the
32-layer model; fewer layers keep the KV pool large enough for B*c = 256K without aliasing).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import (Engine, ModelConfig, Seg, SEG_DECODE, SEG_PREFILL,  # noqa: E402
                                          SEG_FT_FWD, FT_FORWARD, FT_BACKWARD)

P = 16


def make(layers, n_pages, ft_len):
    c = ModelConfig()
    for k, v in bench.L8B.items():
        setattr(c, k, v)
    c.n_layers = layers
    c.norm, c.act, c.rope, c.qkv_bias = 1, 1, 1, 0
    c.rope_theta, c.rms_eps = 500000.0, 1e-5
    c.page_size = P
    c.n_pages = n_pages
    c.max_tokens = 8192
    c.max_ft_len = ft_len
    c.max_segments = 320
    e = Engine(c, device=0)
    e.init_random(1234)
    return e


def timed(eng, fn, reps=5):
    fn()  # warm
    eng.set_profiling(False)
    eng.set_profiling(True)
    ms = []
    for _ in range(reps):
        ms.append(fn())
    prof = {k: eng.read_profile(k) for k in range(4)}
    eng.set_profiling(False)
    return sum(ms) / len(ms), prof


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/kernel_sweep.json")
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    peaks, kind = bench.load_peaks()
    hbm = peaks["hbm_gbs"]
    tc_peak = peaks["bf16_tflops"]
    n_pages = 16384 + 64
    ft_len = 8192
    eng = make(a.layers, n_pages, ft_len)
    res = {"layers": a.layers, "shape": "llama-3.1-8b", "peaks": {"hbm_gbs": hbm, "bf16_tflops": tc_peak,
                                                                  "kind": kind}, "decode": [], "finetune": [], "mixed": []}
    # ---------------------------------------------------------------- decode only
    marks = []  # decode configs in launch order (for the ncu launch-list reduction below)
    Bs = [1, 8, 32, 64, 128, 256]
    Cs = [512, 1024, 2048, 4096, 8192]
    if a.quick:
        Bs, Cs = [64, 256], [1024, 4096]
    for B in Bs:
        for c in Cs:
            per = (c + P) // P + 1
            if B * per > n_pages:
                continue
            pts = [list(range(i * per, (i + 1) * per)) for i in range(B)]
            segs = [Seg(SEG_DECODE, [i % 1000], c, pts[i], sample=False) for i in range(B)]
            ms, prof = timed(eng, lambda: eng.step(segs)["ms"])
            d = prof[1]
            marks.append({"B": B, "ctx": c, "launches": 6 * a.layers,
                          "bytes_per_launch": d["bytes"] / max(1, d["launches"])})
            gbs = d["bytes"] / (d["ms"] * 1e-3) / 1e9 if d["ms"] else 0.0
            row = {"B": B, "ctx": c, "step_ms": round(ms, 3),
                   "attn_us_per_layer": round(d["ms"] * 1e3 / max(1, d["launches"]), 2),
                   "gbs": round(gbs, 1), "hbm_frac": round(gbs / hbm, 4)}
            res["decode"].append(row)
            print("decode", row, flush=True)
    # ---------------------------------------------------------------- finetune only
    ft_pages = list(range(0, ft_len // P))
    toks = [(7 * i) % 1000 for i in range(ft_len)]

    def rate(pr, peak):
        return (round(pr["flops"] / pr["ms"] / 1e9, 1), round(pr["flops"] / pr["ms"] / 1e9 / peak, 4)) \
            if pr["ms"] else (None, None)
    # warm-up: one forward pass and one backward window untimed, so module loading / first-launch
    # costs of the finetuning kernels stay out of the first timed window size (a cold first
    # backward once measured 53 ms for the 1024-token windows instead of 9)
    eng.reset_ft()
    for l in range(0, ft_len, 2048):
        eng.step([Seg(SEG_FT_FWD, toks[l:l + 2048], l, ft_pages, adapter=True)],
                 ft={"phase": FT_FORWARD, "seq_len": ft_len, "l": l, "s": 2048,
                     "targets": toks[l + 1:l + 2049] + ([-1] if l + 2048 == ft_len else [])})
    eng.step([], ft={"phase": FT_BACKWARD, "seq_len": ft_len, "l": ft_len, "s": 2048,
                     "layer": a.layers - 1, "pages": ft_pages})
    for s in ([1024, 2048, 4096] if not a.quick else [2048]):
        eng.reset_ft()
        eng.set_profiling(False)
        eng.set_profiling(True)
        fwd_ms = 0.0
        for l in range(0, ft_len, s):
            fwd_ms += eng.step([Seg(SEG_FT_FWD, toks[l:l + s], l, ft_pages, adapter=True)],
                               ft={"phase": FT_FORWARD, "seq_len": ft_len, "l": l, "s": s,
                                   "targets": toks[l + 1:l + s + 1] + ([-1] if l + s == ft_len else [])})["ms"]
        pf = {k: eng.read_profile(k) for k in range(4)}
        eng.set_profiling(False)
        eng.set_profiling(True)
        bwd_ms = 0.0
        for n in range(a.layers - 1, -1, -1):
            for lj in range(ft_len, 0, -s):
                bwd_ms += eng.step([], ft={"phase": FT_BACKWARD, "seq_len": ft_len, "l": lj, "s": s,
                                           "layer": n, "pages": ft_pages})["ms"]
        pb = {k: eng.read_profile(k) for k in range(4)}
        eng.set_profiling(False)
        eng.reset_ft()
        gf, gff = rate(pf[0], tc_peak)
        af, aff = rate(pf[3], tc_peak)
        gb, gbf = rate(pb[0], tc_peak)
        ab, abf = rate(pb[2], tc_peak)
        row = {"window": s, "seq_len": ft_len, "fwd_ms": round(fwd_ms, 2), "bwd_ms": round(bwd_ms, 2),
               "fwd_gemm_tflops": gf, "fwd_gemm_frac": gff, "fwd_attn_tflops": af, "fwd_attn_frac": aff,
               "bwd_gemm_tflops": gb, "bwd_gemm_frac": gbf, "bwd_attn_tflops": ab, "bwd_attn_frac": abf}
        res["finetune"].append(row)
        print("finetune", row, flush=True)
    # ---------------------------------------------------------------- mixed
    T = 2048
    dec_pages = [list(range(i * 66, i * 66 + 66)) for i in range(64)]
    base = 64 * 66
    fracs = [0, 10, 25, 50, 75, 90, 100] if not a.quick else [0, 50, 100]
    for fr in fracs:
        n_ft = T * fr // 100
        n_inf = T - n_ft
        segs = []
        n_dec = min(64, n_inf)
        segs += [Seg(SEG_DECODE, [i], 1024, dec_pages[i]) for i in range(n_dec)]
        rest = n_inf - n_dec
        pb = base
        while rest > 0:
            w = min(512, rest)
            segs.append(Seg(SEG_PREFILL, toks[:w], 0, list(range(pb, pb + w // P + 1))))
            pb += w // P + 1
            rest -= w
        ftp = list(range(pb, pb + ft_len // P))

        def run():
            eng.reset_ft()
            ss = list(segs)
            ft = None
            if n_ft:
                ss.append(Seg(SEG_FT_FWD, toks[:n_ft], 0, ftp, adapter=True))
                ft = {"phase": FT_FORWARD, "seq_len": ft_len, "l": 0, "s": n_ft,
                      "targets": toks[1:n_ft + 1]}
            return eng.step(ss, ft=ft)["ms"]
        ms, prof = timed(eng, run)
        g = prof[0]
        row = {"ft_pct": fr, "T": T, "step_ms": round(ms, 3),
               "gemm_tflops": round(g["flops"] / g["ms"] / 1e9, 1) if g["ms"] else None,
               "gemm_share": round(g["ms"] / (ms * 5 + 1e-9) if g["ms"] else 0, 3)}
        res["mixed"].append(row)
        print("mixed", row, flush=True)
    res["decode_launch_marks"] = marks
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


def reduce_ncu(sweep_json, launches_csv, out_json):
    """Decode rows of the sweep from ncu device times: `ncu --metrics gpu__time_duration.sum,
    dram__bytes_read.sum -k regex:"attn_decode|attn_combine"` over this script.  Each decode
    config issues 6 steps x layers decode launches (each followed by its combine launch when the
    key ranges were split); the engine's CUDA events time decode-only steps with host launch
    gaps inside, so the roofline fraction is taken from the ncu durations."""
    import csv
    res = json.load(open(sweep_json))
    hdr, per = None, {}
    for r in csv.reader(open(launches_csv)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = per.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
            v = float(d["Metric Value"])
            u = d.get("Metric Unit", "")
            if d["Metric Name"] == "gpu__time_duration.sum":
                e["ns"] = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "nsecond": 1}.get(u, 1)
            else:
                e["bytes"] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    seq = [per[k] for k in sorted(per)]
    # fold each combine into the preceding decode launch
    groups = []
    for e in seq:
        if "attn_decode" in e["name"]:
            groups.append({"ns": e.get("ns", 0.0), "bytes": e.get("bytes", 0.0)})
        elif groups:
            groups[-1]["ns"] += e.get("ns", 0.0)
    hbm = res["peaks"]["hbm_gbs"]
    rows, pos = [], 0
    for m in res["decode_launch_marks"]:
        g = groups[pos:pos + m["launches"]][m["launches"] // 6:]  # drop the warm-up step
        pos += m["launches"]
        if not g:
            break
        ns = sum(x["ns"] for x in g) / len(g)
        gbs = m["bytes_per_launch"] / (ns * 1e-9) / 1e9
        rows.append({"B": m["B"], "ctx": m["ctx"], "kernel_us": round(ns / 1e3, 2),
                     "algorithmic_MB": round(m["bytes_per_launch"] / 1e6, 2),
                     "dram_MB": round(sum(x["bytes"] for x in g) / len(g) / 1e6, 2),
                     "gbs": round(gbs, 1), "hbm_frac": round(gbs / hbm, 4)})
    res["decode_ncu"] = rows
    json.dump(res, open(out_json, "w"), indent=1)
    for r in rows:
        print(r)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--reduce":
        reduce_ncu(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        main()
