import sys, os
sys.path.insert(0, ".")
import numpy as np
from oracle import coserve_oracle as O
import tests.test_coserve_gpu as T
arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
W = O.init_tiny(arch, 1)
toks = list(O.Rng(42).uniform_int(0, 63, 64))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for i in range(n):
    eng, loss_sum, kvg, dys, dmax = T._run_coserve(arch, W, toks, [64], [64], n_inf=2, check_logits=False)
    ga, gb = eng.lora_grads(1)
    print("run", i, "logit diff", dmax, "loss", loss_sum / 63, "gA1 sum", ga.sum(), flush=True)
