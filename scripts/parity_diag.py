"""Print GPU-vs-emu / GPU-vs-f64 / emu-vs-f64 for every gated quantity of the parity configs
(no asserts): localises which stage the GPU departs from the bf16 rounding-point oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import tests.test_coserve_gpu as T  # noqa: E402
from oracle import coserve_oracle as O  # noqa: E402


def table(name, arch, W, toks, fwd, bwd, n_inf=4, kv_layers=(1,)):
    tr, bw, te, be = T.oracles(arch, W, toks)
    eng, loss_sum, kvg, dys, dmax = T._run_coserve(arch, W, toks, fwd, bwd, n_inf=n_inf,
                                                   check_logits=False, test=name)
    print(f"== {name}: loss gpu {loss_sum / (len(toks) - 1):.6f} emu {te['loss']:.6f} f64 {tr['loss']:.6f}")
    rows = []
    for l in range(arch.n_layers):
        ga, gb = eng.lora_grads(l)
        rows += [(f"dA{l}", ga, be["grads"]["a"][l], bw["grads"]["a"][l]),
                 (f"dB{l}", gb, be["grads"]["b"][l], bw["grads"]["b"][l])]
    for n in kv_layers:
        dk, dv = kvg[n]
        rows += [(f"dK{n}", dk, be["layers"][n]["dk"], bw["layers"][n]["dk"]),
                 (f"dV{n}", dv, be["layers"][n]["dv"], bw["layers"][n]["dv"]),
                 (f"dX{n}", dys[n], be["layers"][n]["dx"], bw["layers"][n]["dx"])]
    for q, g, e, f in rows:
        print(f"  {q:5s} gpu-emu {O.scaled_err(g, e):.4f}  gpu-f64 {O.scaled_err(g, f):.4f}  emu-f64 {O.scaled_err(e, f):.4f}")
    eng.close()


which = sys.argv[1:] or ["tiny", "llama", "d128", "qwen"]
if "tiny" in which:
    arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
    W = O.init_tiny(arch, 1)
    toks = list(O.Rng(42).uniform_int(0, 63, 64))
    table("tiny", arch, W, toks, [64], [64])
if "llama" in which:
    arch = T.LLAMA3
    W = O.init_general(arch, 3)
    toks = list(np.random.default_rng(5).integers(0, arch.vocab, 100))
    table("llama", arch, W, toks, [40, 60], [30, 30, 40], n_inf=5, kv_layers=(1, 2))
if "d128" in which:
    arch = T.ARCH_D128
    W = O.init_general(arch, 7)
    toks = list(np.random.default_rng(9).integers(0, arch.vocab, 300))
    table("d128", arch, W, toks, [100, 200], [150, 150], n_inf=5)
if "qwen" in which:
    arch = T.ARCH_QWEN5
    W = O.init_general(arch, 17)
    toks = list(np.random.default_rng(23).integers(0, arch.vocab, 300))
    table("qwen", arch, W, toks, [100, 200], [150, 150], n_inf=5)
