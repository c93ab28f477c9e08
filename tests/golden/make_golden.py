"""Generate tests/golden/*.npz from the reference itself (oracle/_ref/libcoserve_ref.so, the
unmodified reference headers compiled by oracle/Makefile).  Run in the dev container where
/root/reference exists:  python tests/golden/make_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref as R  # noqa: E402


def main():
    assert R.available(), "build oracle/_ref first (make -C oracle)"
    out = {}
    out["rng_mixed_seed5"] = R.rng_mixed(5, 1000)
    out["rng_uniform_int_seed42"] = R.rng_uniform_int(42, 256, 0, 63)
    out["rng_normal_seed7"] = R.rng_normal(7, 512)
    # cfg A (SPEC acceptance config) -- full arrays
    m = R.RefTinyModel(depth=2, hidden=16, heads=1, vocab=64, rank=2, seed=1)
    toks = R.rng_uniform_int(42, 32, 0, 63)
    res = m.forward_backward(toks)
    for k in ("logits", "grad_a", "grad_b", "dk", "dv", "dx", "final_hidden"):
        out["A_" + k] = res[k]
    out["A_loss"] = np.array([res["loss"]])
    out["A_tokens"] = toks
    out["A_embed"] = m.get("embed")
    out["A_lora_b1"] = m.get("lora_b", 1)
    # cfg B (BASELINE tiny config) -- loss, logits, LoRA grads, row sums of dk/dv/dx
    m = R.RefTinyModel(depth=2, hidden=256, heads=4, vocab=64, rank=8, seed=1)
    toks = R.rng_uniform_int(42, 64, 0, 63)
    res = m.forward_backward(toks)
    out["B_loss"] = np.array([res["loss"]])
    out["B_logits"] = res["logits"]
    out["B_grad_a"] = res["grad_a"]
    out["B_grad_b"] = res["grad_b"]
    out["B_dk_rowsum"] = res["dk"].sum(axis=2)
    out["B_dv_rowsum"] = res["dv"].sum(axis=2)
    out["B_dx_rowsum"] = res["dx"].sum(axis=2)
    out["B_dx_l1_row0"] = res["dx"][1, 0]
    out["B_embed00"] = np.array([m.get("embed")[0, 0]])
    out["B_lora_b1_00"] = np.array([m.get("lora_b", 1)[0, 0]])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"))


if __name__ == "__main__":
    main()
