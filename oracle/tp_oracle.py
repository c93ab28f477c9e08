"""Tensor-parallel restatement of the co-serving layer (test infrastructure, CPU only).

SURVEY.md §8e partitioning, which the GPU engine implements (csrc/comm.h, engine.cu):
  * q/k/v heads split over the ranks (QKV column-parallel; rank r owns q heads
    [r*Hq/tp, (r+1)*Hq/tp) and the kv heads they map to), O row-parallel;
  * gate/up columns and down rows split by ffn (column- then row-parallel);
  * LoRA A [f, r] row-sharded with W_down, B [r, h] replicated; the LoRA up-projection
    u_r B is folded into the down partial sum (sum_r (m_r W_r + m_r A_r B) = m W + m A B),
    so the forward needs no extra collective and dB is a per-rank partial reduced once per
    mini-batch (the 'reduce-mid' alternative of test_parallelize.cpp:172-180 all-reduces u);
  * embedding, norms and the LM head replicated.
The per-rank functions are the oracle's own forward/backward (oracle/coserve_oracle.py) run
on the rank's shard with an all-reduce hook `ar` at the exchange points; with tp=1 they are
the single-GPU oracle.  Parity of the sharded math is pinned against the full oracle in
tests/test_tp.py (world-size-2 gloo) -- this file is never on the product path.
"""
from __future__ import annotations

import copy
from typing import Dict, Tuple

import numpy as np

from .coserve_oracle import Arch


def tp_local_arch(arch: Arch, size: int) -> Arch:
    if arch.n_kv_heads % size or arch.n_heads % size or arch.ffn % size:
        raise ValueError("tp size must divide the heads, kv heads and ffn")
    a = copy.copy(arch)
    a.n_heads = arch.n_heads // size
    a.n_kv_heads = arch.n_kv_heads // size
    a.ffn = arch.ffn // size
    return a


def tp_shard(arch: Arch, W: Dict, rank: int, size: int) -> Tuple[Arch, Dict]:
    """(local arch, rank's weights) in the reference layout [in, out]."""
    la = tp_local_arch(arch, size)
    qd, kvd, f = la.q_dim, la.kv_dim, la.ffn
    q = slice(rank * qd, (rank + 1) * qd)
    kv = slice(rank * kvd, (rank + 1) * kvd)
    fs = slice(rank * f, (rank + 1) * f)
    out = {k: v for k, v in W.items() if k != "layers"}
    out["layers"] = []
    for Lw in W["layers"]:
        s = {}
        for k, v in Lw.items():
            if k == "wq":
                s[k] = v[:, q]
            elif k in ("wk", "wv"):
                s[k] = v[:, kv]
            elif k == "bq":
                s[k] = v[q]
            elif k in ("bk", "bv"):
                s[k] = v[kv]
            elif k == "wo":
                s[k] = v[q, :]
            elif k in ("w_gate", "w_up"):
                s[k] = v[:, fs]
            elif k in ("w_down", "lora_a"):
                s[k] = v[fs, :]
            else:  # lora_b, g1, g2: replicated
                s[k] = v
        out["layers"].append(s)
    return la, out
