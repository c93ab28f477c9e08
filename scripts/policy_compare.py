"""Co-serving vs the temporal-sharing baselines of PAPER.md §8.2 on one B200 (8B shape, the
bench's workload): the same engine, profile, trace and SLO; only the scheduling policy
differs (include/coserve/baselines.hpp).

  python scripts/policy_compare.py [--rate 20] [--steps 600] [--out gpurun_out/policies.json]

Finetuning throughput here is the policy-neutral forward-equivalent rate
(fwd tokens + bwd layer-tokens / N) / 2 per second of the timed region, so inference-only
iterations of the temporal policies are charged to it.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_18789_b200.engine import (coserve_run, POLICY_COSERVE, POLICY_TEMPORAL,  # noqa: E402
                                          POLICY_DTS)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, default=20.0)
    ap.add_argument("--steps", type=int, default=600,
                    help="co-serving timed steps; the temporal policies (short inference-only "
                         "steps) get --temporal-mult x as many, for a similar timed duration")
    ap.add_argument("--temporal-mult", type=float, default=5.5)
    ap.add_argument("--warmup", type=int, default=40)
    ap.add_argument("--out", default="gpurun_out/policies.json")
    a = ap.parse_args()
    L = 8192
    n_layers = bench.L8B["n_layers"]
    eng = bench.make_engine(0, L)
    prof = bench.offline_profile(eng, L)
    rows = []
    for name, pol, n in (("coserve", POLICY_COSERVE, 0), ("temporal:64", POLICY_TEMPORAL, 64),
                         ("temporal:128", POLICY_TEMPORAL, 128), ("dts", POLICY_DTS, 0)):
        steps = a.steps if pol == POLICY_COSERVE else int(a.steps * a.temporal_mult)
        c = bench.coserve_config(a.rate, prof, steps, a.warmup, L, seed=7)
        c.policy, c.temporal_n = pol, n
        st, log = coserve_run(eng, c)
        t = st["timed_ms"]
        ft = (st["ft_fwd_tokens"] + st["ft_bwd_tokens"] / n_layers) / 2.0
        row = {"policy": name, "ft_tokens_per_s": round(1000.0 * ft / t, 1),
               "minibatches_done": st["minibatches_done"],
               "gen_tokens_per_s": round(1000.0 * st["gen_tokens"] / t, 1),
               "requests_done": st["requests_done"],
               "slo_attainment": round(st["requests_slo_ok"] / max(1, st["requests_done"]), 4),
               "tpot_p50_ms": round(st["tpot_p50_ms"], 2), "tpot_p99_ms": round(st["tpot_p99_ms"], 2),
               "ttft_p99_ms": round(st["ttft_p99_ms"], 1),
               "iter_p99_ms_inference": round(st["iter_p99_ms"], 2),
               "longest_step_ms": round(max(g["ms"] for g in log if g["timed"]), 1),
               "timed_s": round(t / 1000.0, 2)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    res = {"config": f"LLaMA-3.1-8B-shaped, 1 B200, {a.rate:g} req/s Poisson, TPOT SLO "
                     f"{bench.SLO_MS:g} ms, TTFT SLO 5 s, FT sequences L={L}, max batch {bench.MAX_BATCH}",
           "profile": {k: v for k, v in prof.items() if not k.endswith("samples")},
           "rows": rows}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
