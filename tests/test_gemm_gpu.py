"""K1: tcgen05/TMA GEMM parity vs a torch fp32 reference of the same op (bf16 inputs)."""
import ctypes

import pytest
import torch

from paper_2402_18789_b200 import _lib

pytestmark = pytest.mark.gpu


def _gemm(A, B, C, epi, bias=None, bn=0, splits=0, M=None):
    L = _lib.lib()
    M = A.shape[0] if M is None else M
    N, K = B.shape
    rc = L.cs_gemm_bf16(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(),
                        C.stride(0), M, N, K, epi,
                        None if bias is None else bias.data_ptr(), bn, splits,
                        torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "cs_gemm_bf16")


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 256), (128, 128, 128, 128), (300, 200, 320, 64),
                                      (77, 96, 256, 32), (1000, 1536, 512, 0), (5, 16, 1088, 16),
                                      (4096, 4096, 4096, 0), (64, 6144, 4096, 0),
                                      # CTA-pair (cta_group::2) kernel: >= 74 tiles of 256 x 256
                                      (3000, 4000, 1024, 0), (2048, 28672, 512, 0),
                                      (300, 6144, 1024, 0),
                                      # M <= 64: half-height A stages
                                      (64, 28672, 4096, 0), (17, 6144, 4096, 0), (40, 2048, 576, 0)])
def test_gemm_bf16_out(cuda, M, N, K, bn):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    C = torch.zeros(M, N, device=cuda, dtype=torch.bfloat16)
    _gemm(A, B, C, 0, bn=bn)
    ref = A.float() @ B.float().T
    torch.cuda.synchronize()
    err = (C.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err


@pytest.mark.parametrize("M,N,K,splits", [(128, 256, 1024, 1), (64, 4096, 4096, 0), (256, 512, 2048, 4),
                                          (16, 4096, 14400, 0), (2048, 4096, 4096, 0),
                                          (1500, 4104, 512, 0), (64, 4096, 14400, 0),
                                          (33, 4096, 4096, 0),
                                          (1728, 4096, 14400, 0)])  # CTA pair, tail wave split
def test_gemm_f32_add_splitk(cuda, M, N, K, splits):
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    R = torch.randn(M, N, device=cuda, generator=g)
    C = R.clone()
    _gemm(A, B, C, 2, splits=splits)
    ref = R + A.float() @ B.float().T
    torch.cuda.synchronize()
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-4, err


def test_gemm_f32_store_bias(cuda):
    g = torch.Generator(device="cuda").manual_seed(5)
    M, N, K = 200, 96, 256
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g)
    C = torch.zeros(M, N, device=cuda, dtype=torch.bfloat16)
    _gemm(A, B, C, 0, bias=bias)
    ref = A.float() @ B.float().T + bias
    C2 = torch.full((M, N), 7.0, device=cuda)
    _gemm(A, B, C2, 1, splits=2)
    torch.cuda.synchronize()
    assert (C.float() - ref).abs().max().item() / ref.abs().max().item() < 1e-2
    ref2 = A.float() @ B.float().T
    assert (C2 - ref2).abs().max().item() / ref2.abs().max().item() < 1e-4


def _gemm_mn(A, Bkn, C, epi, bn=0, splits=0):
    """C = A . Bkn with Bkn stored [K, N] (MN-major B operand)."""
    L = _lib.lib()
    M, K = A.shape
    N = Bkn.shape[1]
    rc = L.cs_gemm_bf16_mn(A.data_ptr(), A.stride(0), Bkn.data_ptr(), Bkn.stride(0), C.data_ptr(),
                           C.stride(0), M, N, K, epi, bn, splits,
                           torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "cs_gemm_bf16_mn")


@pytest.mark.parametrize("M,N,K,epi,bn,splits", [
    (128, 256, 64, 0, 256, 0), (300, 200, 320, 0, 64, 0), (1000, 1536, 512, 0, 0, 0),
    (3000, 4096, 1024, 0, 0, 0),          # CTA pair
    (8192, 4096, 28672 // 8, 1, 0, 0),    # dX of gate|up at a full window (K scaled down)
    (640, 4096, 4096, 2, 0, 0),           # mid-M split-K fp32 add
    (1728, 4096, 7168, 2, 0, 0),          # CTA pair, last partial wave split along K
    (64, 6144, 4096, 0, 0, 0), (17, 4096, 4096, 1, 0, 0),   # small M (half-height A)
    (200, 136, 256, 1, 0, 2),             # N tail, forced split
])
def test_gemm_mn_major_b(cuda, M, N, K, epi, bn, splits):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    Bkn = torch.randn(K, N, device=cuda, generator=g).bfloat16()
    if epi == 0:
        C = torch.zeros(M, N, device=cuda, dtype=torch.bfloat16)
        base = 0.0
    else:
        C = torch.randn(M, N, device=cuda, generator=g)
        base = C.clone() if epi == 2 else 0.0
    _gemm_mn(A, Bkn, C, epi, bn=bn, splits=splits)
    ref = base + A.float() @ Bkn.float()
    torch.cuda.synchronize()
    err = (C.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < (1e-2 if epi == 0 else 1e-4), err


@pytest.mark.parametrize("M,f,K", [(64, 1024, 512), (300, 2048, 1024), (2048, 14336, 512), (17, 512, 4096),
                                   (1000, 1536, 512)])
def test_gemm_swiglu_epilogue(cuda, M, f, K):
    """EPI_SWIGLU (the gate||up projection with the SwiGLU fused into the epilogue): B's rows
    interleaved in 64-row [gate | up] blocks; m = silu(bf16 gate) * bf16 up (the unfused path's
    rounding points), the K-concatenation pad columns [f, ldc) zeroed."""
    g = torch.Generator(device="cuda").manual_seed(M + f)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    Wg = torch.randn(f, K, device=cuda, generator=g).bfloat16() / 8
    Wu = torch.randn(f, K, device=cuda, generator=g).bfloat16() / 8
    B = torch.stack([Wg.view(f // 64, 64, K), Wu.view(f // 64, 64, K)], 1).reshape(2 * f, K).contiguous()
    ldc = f + 64
    C = torch.full((M, ldc), 7.0, device=cuda, dtype=torch.bfloat16)
    _gemm(A, B, C, 5)
    gate = (A.float() @ Wg.float().T).bfloat16().float()
    up = (A.float() @ Wu.float().T).bfloat16().float()
    ref = torch.nn.functional.silu(gate) * up
    torch.cuda.synchronize()
    err = (C[:, :f].float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err
    assert C[:, f:].float().abs().max().item() == 0.0


@pytest.mark.parametrize("M,N,K", [(1024, 4096, 32768), (640, 4096, 40960)])
def test_gemm_f32_pair_ksplit(cuda, M, N, K):
    """EPI_F32 with fewer 256 x 256 tiles than CTA pairs and a long K (the LM head's dH): the
    pair kernel with a uniform K split, fp32 atomics into the zeroed output."""
    g = torch.Generator(device="cuda").manual_seed(M + K)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    C = torch.full((M, N), 3.0, device=cuda)
    _gemm(A, B, C, 1)
    ref = A.float() @ B.float().T
    torch.cuda.synchronize()
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-4, err
