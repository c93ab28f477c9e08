// attn_bwd_tc.cu -- K9 on tcgen05 / TMEM: the attention part of a token-level backward window
// (Alg. 2 lines 14-21; tiny_model.hpp:294-315 restricted to query rows
// [a, b) over keys [0, b)).  P is recomputed from Q, K and the saved LSE (no probs stored).
//
// attn_bwd_dq_tc_kernel   : CTA = 128 GQA-packed window rows x 1 KV head, loop over 128-key
//   tiles.  S = Q K^T and dP = dO V^T into TMEM; 8 elementwise warps (one query row per lane,
//   column halves) form dS = P (dP - Delta) in bf16 (K-major SW128 smem); dQ += dS K with K
//   read MN-major straight from its TMA tile.  dQ of the window rows is final.
// attn_bwd_dkdv_tc_kernel : CTA = 128 keys x 1 KV head, loop over 64-row query tiles whose
//   Q / dO arrive by 3-D TMA boxes {64 d, grp heads, 64/grp positions} -- i.e. directly in
//   packed (position, head) order.  S^T = K Q^T, dP^T = V dO^T (double-buffered in TMEM);
//   dV += P^T dO and dK += dS^T Q accumulate in TMEM; the tile's ΔKVAccum rows are owned by
//   the CTA (read-modify-write, no atomics).
#include <atomic>

#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"

namespace cs {

namespace {
constexpr float kLog2eB = 1.4426950408889634f;
constexpr int D = 128;
constexpr int HALF128 = 128 * 128;  // [128 rows][128 B] = 16 KB
constexpr int TILE128 = 2 * HALF128;

CS_DEV uint32_t swz128(int r, int c) {  // chunk c (0..15) of row r, [2 halves][128 rows][128B]
  return (uint32_t)((c >> 3) * HALF128 + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4));
}
CS_DEV uint32_t swz64(int r, int c) {  // chunk c (0..7) of row r, one [rows][128B] atom column
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// paged K/V tile of 128 keys -> two SW128 halves each for K and V (contiguous-run fast path)
CS_DEV void load_kv_tile(const CUtensorMap* tK, const CUtensorMap* tV, const CUtensorMap* tK128,
                         const CUtensorMap* tV128, uint64_t* bar, uint8_t* sk, uint8_t* sv,
                         const int* pt, int page_off, int P, int k0, int k_end, int kvh) {
  const int pg0 = __ldg(pt + page_off + k0 / P);
  bool contig = true;
  for (int key = (k0 / P + 1) * P; key < k0 + 128 && key < k_end; key += P)
    contig &= __ldg(pt + page_off + key / P) == pg0 + (key / P - k0 / P);
  if (contig) {
    const int row = pg0 * P + (k0 % P);
    for (int h = 0; h < 2; ++h) {
      tma_load_2d(tK128, bar, sk + h * HALF128, kvh * D + h * 64, row);
      tma_load_2d(tV128, bar, sv + h * HALF128, kvh * D + h * 64, row);
    }
  } else {
    for (int ch = 0; ch < 8; ++ch) {
      const int key0 = k0 + ch * 16;
      const int row = key0 < k_end ? __ldg(pt + page_off + key0 / P) * P + (key0 % P) : 0;
      for (int h = 0; h < 2; ++h) {
        tma_load_2d(tK, bar, sk + h * HALF128 + ch * 2048, kvh * D + h * 64, row);
        tma_load_2d(tV, bar, sv + h * HALF128 + ch * 2048, kvh * D + h * 64, row);
      }
    }
  }
}
}  // namespace

// ============================================================================ dQ
namespace dq {
constexpr int SMEM_Q = 0;
constexpr int SMEM_O = SMEM_Q + TILE128;
constexpr int SMEM_K = SMEM_O + TILE128;   // 2 stages
constexpr int SMEM_V = SMEM_K + 2 * TILE128;
constexpr int SMEM_DS = SMEM_V + 2 * TILE128;
constexpr int SMEM_BAR = SMEM_DS + TILE128;
constexpr int SMEM_TOTAL = SMEM_BAR + 128 + 1024;
}  // namespace dq

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmK128,
                          const __grid_constant__ CUtensorMap tmV128, AttnBwdParams p) {
  using namespace dq;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
  uint64_t* kv_full = bars + 0;   // [2]
  uint64_t* kv_empty = bars + 2;  // [2]
  uint64_t* s_full = bars + 4;
  uint64_t* s_free = bars + 5;
  uint64_t* ds_full = bars + 6;
  uint64_t* ds_empty = bars + 7;
  uint64_t* q_full = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int grp = p.grp;
  const int rpt = 128 / grp;                // window rows (positions) per CTA
  const int q0 = blockIdx.x * rpt;          // window-local first row
  const int kvh = blockIdx.y;
  const int nq = min(rpt, p.b - p.a - q0);
  const int k_end = p.a + q0 + nq;          // keys [0, last position]
  const int nt = (k_end + 127) / 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmK128);
    tma_prefetch_desc(&tmV128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 256);
    mbar_init(ds_full, 256);
    mbar_init(ds_empty, 1);
    mbar_init(q_full, 256);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < nt; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * TILE128);
        load_kv_tile(&tmK, &tmV, &tmK128, &tmV128, &kv_full[st], smem + SMEM_K + st * TILE128,
                     smem + SMEM_V + st * TILE128, p.page_table, p.page_off, p.page_size, j * 128,
                     k_end, kvh);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idKK = idesc_bf16_f32_major(128, 128, 0, 0);
      constexpr uint32_t idKM = idesc_bf16_f32_major(128, 128, 0, 1);
      const uint32_t sQ = smem_u32(smem + SMEM_Q), sO = smem_u32(smem + SMEM_O);
      const uint32_t sDS = smem_u32(smem + SMEM_DS);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_dq = [&](int jj) {
        const int st = jj & 1;
        mbar_wait(ds_full, jj & 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + SMEM_K + st * TILE128);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = umma_desc_sw128(sDS + (kk >> 2) * HALF128 + (kk & 3) * 32);
          const uint64_t b = umma_desc_sw128_mn(sK + kk * 2048, HALF128, 1024);
          mma_bf16(tmem + 256, a, b, idKM, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&kv_empty[st]);
        mma_commit(ds_empty);
      };
      for (int j = 0; j < nt; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        if (j > 0) mbar_wait(s_free, (j - 1) & 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + SMEM_K + st * TILE128);
        const uint32_t sV = smem_u32(smem + SMEM_V + st * TILE128);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * HALF128 + (kk & 3) * 32;
          mma_bf16(tmem + 0, umma_desc_sw128(sQ + off), umma_desc_sw128(sK + off), idKK, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * HALF128 + (kk & 3) * 32;
          mma_bf16(tmem + 128, umma_desc_sw128(sO + off), umma_desc_sw128(sV + off), idKK, kk > 0);
        }
        mma_commit(s_full);
        if (j > 0) issue_dq(j - 1);
      }
      if (nt > 0) issue_dq(nt - 1);
    }
  } else if (warp >= 4) {
    const int ew = (warp - 4) & 3, hh = (warp - 4) >> 2;
    const int r = ew * 32 + lane;
    const int qr = r / grp, g = r % grp;
    const bool valid = qr < nq;
    const int pos = valid ? p.a + q0 + qr : -1;
    const int qh = kvh * grp + g;
    float lse2 = 0.f, dlt = 0.f;
    {  // Q and dO half rows -> SW128 smem; per-row LSE / Delta in registers
      const bf16* qs = p.q_cache + (long)(valid ? pos : 0) * p.q_ld + (long)qh * D;
      const bf16* os = p.dO + (long)(q0 + (valid ? qr : 0)) * p.do_ld + (long)qh * D;
#pragma unroll
      for (int c = hh * 8; c < hh * 8 + 8; ++c) {
        uint4 vq = make_uint4(0, 0, 0, 0), vo = make_uint4(0, 0, 0, 0);
        if (valid) {
          vq = *reinterpret_cast<const uint4*>(qs + c * 8);
          vo = *reinterpret_cast<const uint4*>(os + c * 8);
        }
        *reinterpret_cast<uint4*>(smem + SMEM_Q + swz128(r, c)) = vq;
        *reinterpret_cast<uint4*>(smem + SMEM_O + swz128(r, c)) = vo;
      }
      if (valid) {
        lse2 = p.lse[(long)pos * p.lse_ld + qh] * kLog2eB;
        dlt = p.delta[(long)(q0 + qr) * p.delta_ld + qh];
      }
      fence_proxy_async_smem();
      mbar_arrive(q_full);
    }
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    for (int j = 0; j < nt; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      uint32_t sv[2][32], dv[2][32];
      tmem_ld_32x32b_x32(tmem + lane_base + hh * 64, sv[0]);
      tmem_ld_32x32b_x32(tmem + lane_base + hh * 64 + 32, sv[1]);
      tmem_ld_32x32b_x32(tmem + lane_base + 128 + hh * 64, dv[0]);
      tmem_ld_32x32b_x32(tmem + lane_base + 128 + hh * 64 + 32, dv[1]);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(s_free);
      const int kb = j * 128 + hh * 64;
      // P = 2^(s*scale*log2e - lse*log2e) (FFMA2 + SFU), dS = P (dP - Delta) (FFMA2 pairs);
      // the causal / k_end mask only on tiles that reach the diagonal
      const bool full = kb + 63 <= pos && kb + 64 <= p.b;
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nl2 = make_float2(-lse2, -lse2);
      const float2 nd2 = make_float2(-dlt, -dlt);
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float2 x = ffma2(make_float2(__uint_as_float(sv[c][i]), __uint_as_float(sv[c][i + 1])), sc2, nl2);
          float2 pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
          if (!full) {
            const int key = kb + c * 32 + i;
            if (!(key <= pos && key < p.b)) pv.x = 0.f;
            if (!(key + 1 <= pos && key + 1 < p.b)) pv.y = 0.f;
          }
          const float2 dd = fadd2(make_float2(__uint_as_float(dv[c][i]), __uint_as_float(dv[c][i + 1])), nd2);
          const float2 d2 = fmul2(pv, dd);
          pk[(c * 32 + i) / 2] = pack_bf16(d2.x, d2.y);
        }
      if (j > 0) {
        mbar_wait(ds_empty, (j - 1) & 1);
        tc_fence_after();
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(smem + SMEM_DS + swz128(r, hh * 8 + c)) =
            make_uint4(pk[c * 4], pk[c * 4 + 1], pk[c * 4 + 2], pk[c * 4 + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(ds_full);
    }
    if (nt > 0) {
      mbar_wait(ds_empty, (nt - 1) & 1);
      tc_fence_after();
    }
    uint32_t o[2][32];
    tmem_ld_32x32b_x32(tmem + lane_base + 256 + hh * 64, o[0]);
    tmem_ld_32x32b_x32(tmem + lane_base + 256 + hh * 64 + 32, o[1]);
    tmem_ld_wait();
    if (valid) {
      float* dst = p.dq + (long)(q0 + qr) * p.dq_ld + (long)qh * D + hh * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + i) =
              make_float4(__uint_as_float(o[c][i]) * p.scale, __uint_as_float(o[c][i + 1]) * p.scale,
                          __uint_as_float(o[c][i + 2]) * p.scale, __uint_as_float(o[c][i + 3]) * p.scale);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================================ dK / dV
namespace kv {
constexpr int QB = 64;                   // packed query rows per tile
constexpr int HALFQ = QB * 128;          // [64 rows][128 B] = 8 KB
constexpr int QTILE = 2 * HALFQ;         // 16 KB
constexpr int SMEM_K = 0;
constexpr int SMEM_V = SMEM_K + TILE128;
constexpr int SMEM_Q = SMEM_V + TILE128;  // 2 stages
constexpr int SMEM_O = SMEM_Q + 2 * QTILE;
constexpr int SMEM_PT = SMEM_O + 2 * QTILE;  // [128 keys][64 rows] bf16 = 16 KB
constexpr int SMEM_DST = SMEM_PT + HALF128;
constexpr int SMEM_X = SMEM_DST + HALF128;   // [2][2][64] floats (lse2, delta)
constexpr int SMEM_BAR = SMEM_X + 2 * 2 * 64 * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
}  // namespace kv

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmK,
                            const __grid_constant__ CUtensorMap tmV,
                            const __grid_constant__ CUtensorMap tmK128,
                            const __grid_constant__ CUtensorMap tmV128,
                            const __grid_constant__ CUtensorMap tmQ3,
                            const __grid_constant__ CUtensorMap tmO3, AttnBwdParams p) {
  using namespace kv;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;    // [2]
  uint64_t* q_empty = bars + 3;   // [2]
  uint64_t* st_full = bars + 5;   // [2]
  uint64_t* st_free = bars + 7;   // [2]
  uint64_t* pds_full = bars + 9;
  uint64_t* pds_empty = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  float* xch = reinterpret_cast<float*>(smem + SMEM_X);

  const int grp = p.grp;
  const int rpt = QB / grp;                // positions per query tile
  const int k0 = blockIdx.x * 128;
  const int kvh = blockIdx.y;
  const int nrows = p.b - p.a;
  const int n_qt = (nrows + rpt - 1) / rpt;
  const int qt0 = k0 > p.a ? (k0 - p.a) / rpt : 0;  // first tile whose last position >= k0
  const int n = n_qt - qt0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ3);
    tma_prefetch_desc(&tmO3);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&st_full[i], 1);
      mbar_init(&st_free[i], 256);
    }
    mbar_init(pds_full, 256);
    mbar_init(pds_empty, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S^T[2] @0,64 ; dP^T[2] @128,192 ; dV @256 ; dK @384

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * TILE128);
      load_kv_tile(&tmK, &tmV, &tmK128, &tmV128, kv_full, smem + SMEM_K, smem + SMEM_V,
                   p.page_table, p.page_off, p.page_size, k0, p.b, kvh);
      for (int i = 0; i < n; ++i) {
        const int st = i & 1;
        const int qt = qt0 + i;
        mbar_wait(&q_empty[st], ((i >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[st], 2 * QTILE);
        for (int h = 0; h < 2; ++h) {
          tma_load_3d(&tmQ3, &q_full[st], smem + SMEM_Q + st * QTILE + h * HALFQ, h * 64, kvh * grp,
                      p.a + qt * rpt);
          tma_load_3d(&tmO3, &q_full[st], smem + SMEM_O + st * QTILE + h * HALFQ, h * 64, kvh * grp,
                      qt * rpt);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32_major(128, QB, 0, 0);
      constexpr uint32_t idG = idesc_bf16_f32_major(128, 128, 0, 1);
      const uint32_t sK = smem_u32(smem + SMEM_K), sV = smem_u32(smem + SMEM_V);
      const uint32_t sPT = smem_u32(smem + SMEM_PT), sDST = smem_u32(smem + SMEM_DST);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      auto issue_grad = [&](int ii) {
        const int st = ii & 1;
        mbar_wait(pds_full, ii & 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + SMEM_Q + st * QTILE);
        const uint32_t sO = smem_u32(smem + SMEM_O + st * QTILE);
#pragma unroll
        for (int kk = 0; kk < QB / 16; ++kk) {
          mma_bf16(tmem + 256, umma_desc_sw128(sPT + kk * 32),
                   umma_desc_sw128_mn(sO + kk * 2048, HALFQ, 1024), idG, (ii > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < QB / 16; ++kk) {
          mma_bf16(tmem + 384, umma_desc_sw128(sDST + kk * 32),
                   umma_desc_sw128_mn(sQ + kk * 2048, HALFQ, 1024), idG, (ii > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&q_empty[st]);
        mma_commit(pds_empty);
      };
      for (int i = 0; i < n; ++i) {
        const int st = i & 1;
        mbar_wait(&q_full[st], (i >> 1) & 1);
        mbar_wait(&st_free[st], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + SMEM_Q + st * QTILE);
        const uint32_t sO = smem_u32(smem + SMEM_O + st * QTILE);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ak = (kk >> 2) * HALF128 + (kk & 3) * 32;
          const uint32_t bq = (kk >> 2) * HALFQ + (kk & 3) * 32;
          mma_bf16(tmem + st * 64, umma_desc_sw128(sK + ak), umma_desc_sw128(sQ + bq), idS, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ak = (kk >> 2) * HALF128 + (kk & 3) * 32;
          const uint32_t bq = (kk >> 2) * HALFQ + (kk & 3) * 32;
          mma_bf16(tmem + 128 + st * 64, umma_desc_sw128(sV + ak), umma_desc_sw128(sO + bq), idS, kk > 0);
        }
        mma_commit(&st_full[st]);
        if (i > 0) issue_grad(i - 1);
      }
      if (n > 0) issue_grad(n - 1);
    }
  } else if (warp >= 4) {
    const int ew = (warp - 4) & 3, hh = (warp - 4) >> 2;  // hh: 32-column half of the 64
    const int t = threadIdx.x - 128;                      // 0..255
    const int key = k0 + ew * 32 + lane;                  // TMEM lane == key row
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    int cq[32];  // position offset (within a query tile) of this thread's 32 packed columns
#pragma unroll
    for (int j = 0; j < 32; ++j) cq[j] = (hh * 32 + j) / grp;
    for (int i = 0; i < n; ++i) {
      const int st = i & 1;
      const int qt = qt0 + i;
      // per-column (packed query row) log2-LSE and Delta for this tile
      float* xs = xch + (i & 1) * 128;
      if (t < 128) {
        const int col = t & 63;
        const int qr = qt * rpt + col / grp, g = col % grp;
        float v = 0.f;
        if (qr < nrows) {
          if (t < 64) v = p.lse[(long)(p.a + qr) * p.lse_ld + kvh * grp + g] * kLog2eB;
          else v = p.delta[(long)qr * p.delta_ld + kvh * grp + g];
        }
        xs[t] = v;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mbar_wait(&st_full[st], (i >> 1) & 1);
      tc_fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld_32x32b_x32(tmem + lane_base + st * 64 + hh * 32, sv);
      tmem_ld_32x32b_x32(tmem + lane_base + 128 + st * 64 + hh * 32, dv);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&st_free[st]);
      uint32_t pp[16], pd[16];
      // column c is query position a + qt*rpt + cq[c]: the tile is fully unmasked for this key
      // when key <= its first position and every column is a real row
      const int qbase = qt * rpt;
      const bool full = key < p.b && key <= p.a + qbase && qbase + cq[31] < nrows;
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const int col = hh * 32 + j;
        float2 x = ffma2(make_float2(__uint_as_float(sv[j]), __uint_as_float(sv[j + 1])), sc2,
                         make_float2(-xs[col], -xs[col + 1]));
        float2 pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        if (!full) {
          const int q0r = qbase + cq[j], q1r = qbase + cq[j + 1];
          if (!(q0r < nrows && key <= p.a + q0r && key < p.b)) pv.x = 0.f;
          if (!(q1r < nrows && key <= p.a + q1r && key < p.b)) pv.y = 0.f;
        }
        const float2 dd = fadd2(make_float2(__uint_as_float(dv[j]), __uint_as_float(dv[j + 1])),
                                make_float2(-xs[64 + col], -xs[64 + col + 1]));
        const float2 ds = fmul2(pv, dd);
        pp[j / 2] = pack_bf16(pv.x, pv.y);
        pd[j / 2] = pack_bf16(ds.x, ds.y);
      }
      if (i > 0) {
        mbar_wait(pds_empty, (i - 1) & 1);
        tc_fence_after();
      }
      const int r = ew * 32 + lane;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        *reinterpret_cast<uint4*>(smem + SMEM_PT + swz64(r, hh * 4 + c)) =
            make_uint4(pp[c * 4], pp[c * 4 + 1], pp[c * 4 + 2], pp[c * 4 + 3]);
        *reinterpret_cast<uint4*>(smem + SMEM_DST + swz64(r, hh * 4 + c)) =
            make_uint4(pd[c * 4], pd[c * 4 + 1], pd[c * 4 + 2], pd[c * 4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(pds_full);
    }
    if (n > 0) {
      mbar_wait(pds_empty, (n - 1) & 1);
      tc_fence_after();
    }
    // ΔKVAccum rows [k0, k0+128) of this head: 64 columns of dV and dK per thread
    uint32_t a0[32], a1[32];
    tmem_ld_32x32b_x32(tmem + lane_base + 256 + hh * 64, a0);
    tmem_ld_32x32b_x32(tmem + lane_base + 256 + hh * 64 + 32, a1);
    tmem_ld_wait();
    if (key < p.b && n > 0) {
      float* av = p.dv_acc + (long)key * p.acc_ld + kvh * D + hh * 64;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 x = *reinterpret_cast<float4*>(av + i);
        x.x += __uint_as_float(a0[i]); x.y += __uint_as_float(a0[i + 1]);
        x.z += __uint_as_float(a0[i + 2]); x.w += __uint_as_float(a0[i + 3]);
        *reinterpret_cast<float4*>(av + i) = x;
        float4 y = *reinterpret_cast<float4*>(av + 32 + i);
        y.x += __uint_as_float(a1[i]); y.y += __uint_as_float(a1[i + 1]);
        y.z += __uint_as_float(a1[i + 2]); y.w += __uint_as_float(a1[i + 3]);
        *reinterpret_cast<float4*>(av + 32 + i) = y;
      }
    }
    tmem_ld_32x32b_x32(tmem + lane_base + 384 + hh * 64, a0);
    tmem_ld_32x32b_x32(tmem + lane_base + 384 + hh * 64 + 32, a1);
    tmem_ld_wait();
    if (key < p.b && n > 0) {
      float* ak = p.dk_acc + (long)key * p.acc_ld + kvh * D + hh * 64;
      const float sc = p.scale;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 x = *reinterpret_cast<float4*>(ak + i);
        x.x += __uint_as_float(a0[i]) * sc; x.y += __uint_as_float(a0[i + 1]) * sc;
        x.z += __uint_as_float(a0[i + 2]) * sc; x.w += __uint_as_float(a0[i + 3]) * sc;
        *reinterpret_cast<float4*>(ak + i) = x;
        float4 y = *reinterpret_cast<float4*>(ak + 32 + i);
        y.x += __uint_as_float(a1[i]) * sc; y.y += __uint_as_float(a1[i + 1]) * sc;
        y.z += __uint_as_float(a1[i + 2]) * sc; y.w += __uint_as_float(a1[i + 3]) * sc;
        *reinterpret_cast<float4*>(ak + 32 + i) = y;
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// single-kernel launchers (A/B against attn_bwd2.cu)
void attn_bwd_dq_v1(const AttnBwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                    const CUtensorMap& tmK128, const CUtensorMap& tmV128, dim3 grid, cudaStream_t st) {
  static bool once = (cudaFuncSetAttribute(attn_bwd_dq_tc_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, dq::SMEM_TOTAL),
                      true);
  (void)once;
  attn_bwd_dq_tc_kernel<<<grid, 384, dq::SMEM_TOTAL, st>>>(tmK, tmV, tmK128, tmV128, p);
}
void attn_bwd_dkdv_v1(const AttnBwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                      const CUtensorMap& tmK128, const CUtensorMap& tmV128, const CUtensorMap& tmQ3,
                      const CUtensorMap& tmO3, dim3 grid, cudaStream_t st) {
  static bool once = (cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kv::SMEM_TOTAL),
                      true);
  (void)once;
  attn_bwd_dkdv_tc_kernel<<<grid, 384, kv::SMEM_TOTAL, st>>>(tmK, tmV, tmK128, tmV128, tmQ3, tmO3, p);
}

// ============================================================================ launcher
cudaError_t attn_bwd_tc(const AttnBwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                        const CUtensorMap& tmK128, const CUtensorMap& tmV128,
                        const CUtensorMap& tmQ3, const CUtensorMap& tmO3, int n_heads,
                        cudaStream_t st) {
  const int rows = p.b - p.a;
  if (rows <= 0) return cudaSuccess;
  static bool once = (cudaFuncSetAttribute(attn_bwd_dq_tc_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           dq::SMEM_TOTAL),
                      cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kv::SMEM_TOTAL),
                      true);
  (void)once;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  attn_bwd_delta_kernel_launch(p, rows, n_heads, st);
  const int kvh = n_heads / p.grp;
  dim3 gq((rows + 128 / p.grp - 1) / (128 / p.grp), kvh);
  dim3 gk((p.b + 127) / 128, kvh);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  attn_bwd_dq_tc_kernel<<<gq, 384, dq::SMEM_TOTAL, st>>>(tmK, tmV, tmK128, tmV128, p);
  attn_bwd_dkdv_tc_kernel<<<gk, 384, kv::SMEM_TOTAL, st>>>(tmK, tmV, tmK128, tmV128, tmQ3, tmO3, p);
  return cudaGetLastError();
}

}  // namespace cs
