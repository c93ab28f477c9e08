"""Print the backward parity errors of the d=128 test scenario for the current attention
backward kernel selection (CS_ATTN_BWD2 / CS_ATTN_TC env)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from oracle import coserve_oracle as O  # noqa: E402
from tests.test_coserve_gpu import ARCH_D128, _run_coserve  # noqa: E402

arch = ARCH_D128
W = O.init_general(arch, 7)
toks = list(np.random.default_rng(9).integers(0, arch.vocab, 300))
tr = O.forward_full(arch, W, toks)
bw = O.backward_full(arch, W, tr)
for wins in ([150, 150], [300], [100, 200]):
    eng, loss_sum, kvg, dys, dmax = _run_coserve(arch, W, toks, [100, 200], wins, n_inf=5,
                                                 logit_tol=1.0)
    dk, dv = kvg[1]
    out = {"wins": wins, "dk": O.scaled_err(dk, bw["layers"][1]["dk"]),
           "dv": O.scaled_err(dv, bw["layers"][1]["dv"]),
           "dx": O.scaled_err(dys[1], bw["layers"][1]["dx"])}
    for l in range(arch.n_layers):
        ga, gb = eng.lora_grads(l)
        out[f"dA{l}"] = O.scaled_err(ga, bw["grads"]["a"][l])
    # per-row error profile of dk (which rows are off)
    err = np.abs(dk - bw["layers"][1]["dk"]).max(axis=1) / np.abs(bw["layers"][1]["dk"]).max()
    out["dk_worst_rows"] = [int(i) for i in np.argsort(-err)[:8]]
    print(os.environ.get("CS_ATTN_BWD2", "1"), {k: (round(v, 4) if isinstance(v, float) else v)
                                                 for k, v in out.items()}, flush=True)
    eng.close()
