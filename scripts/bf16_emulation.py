"""Emulate the GPU path's bf16 rounding points on the reference arch (numpy, CPU) and
report the resulting LoRA-grad / dX errors vs the f64 oracle: the precision floor the GPU
numbers should be compared against."""
import sys
sys.path.insert(0, ".")
import math
import numpy as np
import torch
from oracle import coserve_oracle as O

def bf(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).bfloat16().float().numpy().astype(np.float64)

arch = O.Arch.reference(depth=2, hidden=256, heads=4, vocab=64, rank=8)
W = O.init_tiny(arch, 1)
toks = np.array(list(O.Rng(42).uniform_int(0, 63, 64)))
L, H, d = 64, 4, 64
tr = O.forward_full(arch, W, list(toks))
bw = O.backward_full(arch, W, tr)
Wb = {"embed": bf(W["embed"]), "unembed": bf(W["unembed"]),
      "layers": [{k: (bf(v) if k not in ("lora_a", "lora_b") else v) for k, v in Lw.items()} for Lw in W["layers"]]}
scale = 1 / math.sqrt(d)
mask = np.tril(np.ones((L, L), bool))
def attn(q, k, v):
    out = np.zeros_like(q); lse = np.zeros((L, H))
    for h in range(H):
        s = (q[:, h*d:(h+1)*d] @ k[:, h*d:(h+1)*d].T) * scale
        s = np.where(mask, s, -np.inf); mx = s.max(1, keepdims=True); p = np.exp(s - mx); den = p.sum(1, keepdims=True)
        lse[:, h] = (mx + np.log(den))[:, 0]
        out[:, h*d:(h+1)*d] = bf(p) @ v[:, h*d:(h+1)*d] / den
    return out, lse
x = Wb["embed"][toks].copy()
sav = []
for l in range(2):
    w = Wb["layers"][l]
    xb = bf(x)
    q, k, v = bf(xb @ w["wq"]), bf(xb @ w["wk"]), bf(xb @ w["wv"])
    a, lse = attn(q, k, v); a = bf(a)
    r1 = x + a @ w["wo"]
    up = bf(bf(r1) @ w["w_up"]); m = np.maximum(up, 0)
    lu = m @ bf(w["lora_a"])
    x = r1 + m @ w["w_down"] + bf(lu) @ bf(w["lora_b"])
    sav.append(dict(q=q, k=k, v=v, a=a, lse=lse, up=up, m=m, lu=lu))
logits = bf(x) @ Wb["unembed"]
dlog = np.zeros_like(logits)
for i in range(L - 1):
    e = np.exp(logits[i] - logits[i].max()); dlog[i] = e / e.sum() / (L - 1); dlog[i, toks[i+1]] -= 1 / (L - 1)
Y = bf(dlog) @ Wb["unembed"].T
res = {}
for l in (1, 0):
    w = Wb["layers"][l]; s = sav[l]
    B = W["layers"][l]["lora_b"]; A = W["layers"][l]["lora_a"]
    dlu = Y @ B.T
    gB = s["lu"].T @ Y; gA = s["m"].T @ dlu
    res[l] = (gA, gB)
    if l == 0: break
    dm = bf(Y) @ w["w_down"].T + bf(dlu) @ bf(A).T
    dup = bf(np.where(s["m"] > 0, dm, 0))
    dr1 = Y + dup @ w["w_up"].T
    dO = bf(bf(dr1) @ w["wo"].T)
    dq = np.zeros((L, 256)); dk = np.zeros((L, 256)); dv = np.zeros((L, 256))
    for h in range(H):
        sl = slice(h*d, (h+1)*d)
        sc = np.where(mask, (s["q"][:, sl] @ s["k"][:, sl].T) * scale, -np.inf)
        p = np.exp(sc - s["lse"][:, h:h+1])
        dp = dO[:, sl] @ s["v"][:, sl].T
        delta = (dO[:, sl] * s["a"][:, sl]).sum(1, keepdims=True)
        ds = p * (dp - delta)
        dq[:, sl] = bf(ds) @ s["k"][:, sl] * scale
        dk[:, sl] = bf(ds).T @ s["q"][:, sl] * scale
        dv[:, sl] = bf(p).T @ dO[:, sl]
    dx = dr1 + bf(dq) @ w["wq"].T + bf(dk) @ w["wk"].T + bf(dv) @ w["wv"].T
    print("emulated dk1", O.scaled_err(dk, bw["layers"][1]["dk"]), "dv1", O.scaled_err(dv, bw["layers"][1]["dv"]), "dx1", O.scaled_err(dx, bw["layers"][1]["dx"]))
    Y = dx
for l in (0, 1):
    print("emulated layer", l, "gA", O.scaled_err(res[l][0], bw["grads"]["a"][l]), "gB", O.scaled_err(res[l][1], bw["grads"]["b"][l]))
