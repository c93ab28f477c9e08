// attn_dq_gemm.cu -- dQ of a token-level backward window as a masked GEMM over the dS the
// dK/dV kernel already computed (CS_BWD_DSQ=1): dQ[p, h, :] = scale * sum_k dS[p, h, k] K[k, :]
// (tiny_model.hpp:294-315, Alg. 2 line 19).  The dK/dV kernel holds dS^T in TMEM for
// its own dK product; it also stores it (bf16) as [kv head][64-row query tile][8-row chunk]
// [key][8 rows] -- a warp's 32 keys write 512 contiguous bytes per chunk -- and this kernel
// streams it back as a no-swizzle MN-major A operand (two 64-row tiles per 128-row dQ tile,
// {8 rows, 64 keys, 8 chunks} TMA boxes) against the paged K tile as an MN-major B operand.  It
// replaces the dQ kernel that recomputed S and dP and was bounded by reading both back out of
// TMEM (128 KB per 128x128 tile at 64 B/clk).
//   warp 0: TMA producer (A: 3-D dS box, B: paged K rows, contiguous pages in one 64-row box)
//   warp 1: single-thread tcgen05.mma M=128 N=128 (A K-major, B MN-major), fp32 in TMEM
//   warps 4-7: epilogue (tcgen05.ld, scale, fp32 dQ rows of the window)
#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"

namespace cs {

namespace {
// two 128-row dQ tiles per CTA share every K stage (M = 256 in two TMEM accumulators): half the
// K-tile traffic and half the CTAs of one tile per CTA
constexpr int DQG_TPC = 2;
constexpr int DQG_STAGES = 4;
constexpr int DQG_A1 = 128 * 128;     // one dQ tile: 64 keys x 128 packed rows x bf16 (two 8 KB boxes)
constexpr int DQG_A = DQG_TPC * DQG_A1;
constexpr int DQG_B = 64 * 128 * 2;   // 64 keys x 128 dims x bf16 (two 64-dim chunks, 8 KB apart)
constexpr int DQG_STAGE = DQG_A + DQG_B;
constexpr int DQG_SMEM = DQG_STAGES * DQG_STAGE + 1024 + 256;
// no-swizzle MN-major A (dS^T): core matrices of 8 keys x 8 rows; K-adjacent ones 128 B apart,
// MN-adjacent ones (next 8 rows) 1 KB apart
// (LBO = the K-direction stride, SBO = the MN-direction stride for no-swizzle MN-major
// operands -- the opposite of the SW128 MN-major convention; the swapped assignment fails the
// dS-GEMM parity test)
constexpr uint32_t kDsLbo = 128, kDsSbo = 1024;
}  // namespace

__global__ void __launch_bounds__(256, 1)
    attn_dq_gemm_kernel(const __grid_constant__ CUtensorMap tmDS, const __grid_constant__ CUtensorMap tmK16,
                        const __grid_constant__ CUtensorMap tmK64, AttnBwdParams p, int Hq) {
  griddep_launch();
  griddep_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DQG_STAGES * DQG_STAGE);
  uint64_t* empty = full + DQG_STAGES;
  uint64_t* acc_full = empty + DQG_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int grp = p.grp;
  const int rpt = 128 / grp;  // positions per tile (rpt * grp <= 128 packed rows)
  const int rows = p.b - p.a;
  // longest tiles first (causal: a tile's key range grows with its position), so the last wave
  // holds the short ones
  const int qt0 = (gridDim.x - 1 - blockIdx.x) * DQG_TPC;
  const int kvh = blockIdx.y;
  int nq[DQG_TPC], nkb[DQG_TPC];
  int nkb_max = 0;
#pragma unroll
  for (int t = 0; t < DQG_TPC; ++t) {
    nq[t] = min(rpt, rows - (qt0 + t) * rpt);  // <= 0: no such tile (the window's end)
    nkb[t] = nq[t] > 0 ? (p.a + (qt0 + t) * rpt + nq[t] - 1 + 64) / 64 : 0;  // causal key blocks
    nkb_max = max(nkb_max, nkb[t]);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmDS);
    tma_prefetch_desc(&tmK16);
    tma_prefetch_desc(&tmK64);
    for (int s = 0; s < DQG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 128 * DQG_TPC);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nkb_max; ++kb) {
      const int s = kb % DQG_STAGES;
      mbar_wait(&empty[s], ((kb / DQG_STAGES) & 1) ^ 1);
      int act = 0;
#pragma unroll
      for (int t = 0; t < DQG_TPC; ++t) act += kb < nkb[t];
      mbar_arrive_expect_tx(&full[s], act * DQG_A1 + DQG_B);
      uint8_t* sa = smem + s * DQG_STAGE;
      uint8_t* sb = sa + DQG_A;
      // each dQ tile's two 64-row dK/dV tiles: {8 rows, 64 keys, 8 chunks} boxes, 8 KB each,
      // land as [16 chunks][64 keys][8 rows] -- uniform core-matrix strides over both.  A tile
      // past its causal key range is not loaded (its dS there was never written)
#pragma unroll
      for (int t = 0; t < DQG_TPC; ++t)
        if (kb < nkb[t])
          for (int m = 0; m < 2; ++m)
            tma_load_3d(&tmDS, &full[s], sa + t * DQG_A1 + m * 8192, 0, kb * 64,
                        (int)(((long)kvh * p.ds_heads + 2 * (qt0 + t) + m) * 8));
      // K rows [kb*64, kb*64+64) of the sequence: one 64-row box per 64-dim half when the four
      // 16-key pages are consecutive in the pool, else one 16-row box per page
      const int k0 = kb * 64, P = p.page_size;
      const int pg0 = __ldg(p.page_table + p.page_off + k0 / P);
      bool contig = (P % 16) == 0;
      for (int key = (k0 / P + 1) * P; contig && key < k0 + 64; key += P)
        contig = __ldg(p.page_table + p.page_off + key / P) == pg0 + (key / P - k0 / P);
      for (int c = 0; c < 2; ++c) {
        const int col = kvh * 128 + c * 64;
        if (contig) {
          tma_load_2d(&tmK64, &full[s], sb + c * 8192, col, pg0 * P + (k0 % P));
        } else {
          for (int j = 0; j < 4; ++j) {
            const int key = k0 + 16 * j;
            const int row = __ldg(p.page_table + p.page_off + key / P) * P + (key % P);
            tma_load_2d(&tmK16, &full[s], sb + c * 8192 + j * 2048, col, row);
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32_major(128, 128, 1, 1);  // A and B MN-major
    for (int kb = 0; kb < nkb_max; ++kb) {
      const int s = kb % DQG_STAGES;
      mbar_wait(&full[s], (kb / DQG_STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * DQG_STAGE), sb = sa + DQG_A;
#pragma unroll
      for (int t = 0; t < DQG_TPC; ++t) {
        if (kb >= nkb[t]) continue;
#pragma unroll
        for (int k = 0; k < 4; ++k)  // A: 16 keys = two 128-byte core matrices along K
          mma_bf16(tmem + t * 128, umma_desc_plain(sa + t * DQG_A1 + k * 256, kDsLbo, kDsSbo),
                   umma_desc_sw128_mn(sb + k * 2048, 8192, 1024), idesc, (kb > 0 || k > 0) ? 1u : 0u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(acc_full);
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int r = ew * 32 + lane;  // packed row = TMEM lane
    const int qr = r / grp, g = r - qr * grp;
    mbar_wait(acc_full, 0);
    tc_fence_after();
#pragma unroll 1
    for (int t = 0; t < DQG_TPC; ++t) {
      const bool valid = qr < nq[t] && r < rpt * grp;
      const uint32_t tb = tmem + ((uint32_t)(ew * 32) << 16) + t * 128;
      float* dst = p.dq + (long)((qt0 + t) * rpt + (valid ? qr : 0)) * p.dq_ld + (long)(kvh * grp + g) * 128;
      if (nq[t] <= 0) continue;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tb + c0, v);
        tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + c0 + i) =
                make_float4(__uint_as_float(v[i]) * p.scale, __uint_as_float(v[i + 1]) * p.scale,
                            __uint_as_float(v[i + 2]) * p.scale, __uint_as_float(v[i + 3]) * p.scale);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 128 * DQG_TPC);
  }
}

cudaError_t attn_dq_gemm(const AttnBwdParams& p, const CUtensorMap& tmDS, const CUtensorMap& tmK16,
                         const CUtensorMap& tmK64, int n_heads, cudaStream_t st) {
  const int rows = p.b - p.a;
  if (rows <= 0) return cudaSuccess;
  static bool once = (cudaFuncSetAttribute(attn_dq_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           DQG_SMEM),
                      true);
  (void)once;
  const int rpt = 128 / p.grp;
  const int tiles = (rows + rpt - 1) / rpt;
  dim3 grid((tiles + DQG_TPC - 1) / DQG_TPC, n_heads / p.grp);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return launch_pdl(attn_dq_gemm_kernel, grid, dim3(256), DQG_SMEM, st, tmDS, tmK16, tmK64, p, n_heads);
}

}  // namespace cs
