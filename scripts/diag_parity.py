import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import coserve_oracle as O
import tests.test_coserve_gpu as T

arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
W = O.init_tiny(arch, 1)
toks = list(O.Rng(42).uniform_int(0, 63, 64))
tr = O.forward_full(arch, W, toks)
bw = O.backward_full(arch, W, tr)
for fw, bwin in [([64], [64]), ([20, 44], [64]), ([64], [32, 32])]:
    eng, loss_sum, kvg, dys, dmax = T._run_coserve(arch, W, toks, fw, bwin, n_inf=2, check_logits=False)
    print("windows", fw, bwin, "logit diff", dmax, "loss", loss_sum / 63, tr["loss"])
    for l in range(2):
        ga, gb = eng.lora_grads(l)
        print(" layer", l, "gA", T._errs(ga, bw["grads"]["a"][l]), "gB", T._errs(gb, bw["grads"]["b"][l]))
    dk, dv = kvg[1]
    print(" dk1", O.scaled_err(dk, bw["layers"][1]["dk"]), "dv1", O.scaled_err(dv, bw["layers"][1]["dv"]), "dx1", O.scaled_err(dys[1], bw["layers"][1]["dx"]))
    dx = dys[1]; ref = bw["layers"][1]["dx"]
    print("  dx rows err", np.abs(dx-ref).max(axis=1)[:8], np.abs(ref).max())
    print("  dk rows err", np.abs(dk-bw["layers"][1]["dk"]).max(axis=1)[::8])
