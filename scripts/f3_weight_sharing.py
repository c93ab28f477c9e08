"""SURVEY §8f row 3 (forward / backward weight-tile sharing, the B200 stand-in for the paper's
two-stream space sharing): how much could streaming one layer's frozen weights ONCE for both its
forward products (x W) and its backward dX products (dY W^T) save, at the weight-bound operating
points (T <= ~300 rows)?

For the LLaMA-8B layer (QKV, O, gate||up, down) at T rows: time of the forward GEMMs alone, of
the backward dX GEMMs alone (the MN-major reads of the same weights), and of both back to back
(CUDA events, L2 flushed between repetitions).  A fused kernel sharing each weight tile between
the two products can at best hide one of the two weight streams: saving <= min(t_fwd, t_bwd)
per layer and iteration -- and a co-serving iteration runs the backward window of ONE layer, so
that bound applies once per iteration, next to the ~45 ms SLO-filled iteration.

    python scripts/f3_weight_sharing.py [T ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_18789_b200 import _lib  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
h, f, qkv = 4096, 14336, 6144
W = {"qkv": torch.randn(qkv, h, device=dev).bfloat16(), "o": torch.randn(h, h, device=dev).bfloat16(),
     "gu": torch.randn(2 * f, h, device=dev).bfloat16(), "down": torch.randn(h, f, device=dev).bfloat16()}
st = torch.cuda.current_stream().cuda_stream


def gemm(A, B, C, M, N, K, epi, mn=False):
    if mn:  # C[M, N] = A[M, K] . B  with B stored [K][N] (the forward weight read MN-major)
        rc = L.cs_gemm_bf16_mn(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(), C.stride(0),
                               M, N, K, epi, 0, 0, st)
    else:
        rc = L.cs_gemm_bf16(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(), C.stride(0),
                            M, N, K, epi, None, 0, 0, st)
    _lib.check(rc, "gemm")


def timed(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for T in [int(x) for x in (sys.argv[1:] or ["64", "128", "256", "512", "2048"])]:
    x = torch.randn(T, h, device=dev).bfloat16()
    m = torch.randn(T, f, device=dev).bfloat16()
    a = torch.randn(T, h, device=dev).bfloat16()
    out = {k: torch.empty(T, W[k].shape[0], device=dev, dtype=torch.bfloat16) for k in W}
    dy = {k: torch.randn(T, W[k].shape[0], device=dev).bfloat16() for k in W}
    dx = {k: torch.empty(T, W[k].shape[1], device=dev, dtype=torch.bfloat16) for k in W}

    def fwd():
        gemm(x, W["qkv"], out["qkv"], T, qkv, h, 0)
        gemm(a, W["o"], out["o"], T, h, h, 0)
        gemm(x, W["gu"], out["gu"], T, 2 * f, h, 0)
        gemm(m, W["down"], out["down"], T, h, f, 0)

    def bwd():  # dX = dY W^T: the forward [out, in] copy read MN-major
        for k in W:
            N_out, K_in = W[k].shape
            gemm(dy[k], W[k], dx[k], T, K_in, N_out, 0, mn=True)

    tf, tb = timed(fwd), timed(bwd)
    tfb = timed(lambda: (fwd(), bwd()))
    wbytes = sum(w.numel() * 2 for w in W.values())
    print(json.dumps({"T": T, "fwd_ms": round(tf, 4), "bwd_dx_ms": round(tb, 4), "both_ms": round(tfb, 4),
                      "weight_MB": round(wbytes / 1e6, 1),
                      "weight_stream_ms_at_hbm": round(wbytes / 6.5e12 * 1e3, 4),
                      "sharing_upper_bound_ms": round(min(tf, tb), 4),
                      "bound_pct_of_45ms_iteration": round(100 * min(tf, tb) / 45.0, 2)}), flush=True)
