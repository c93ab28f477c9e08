// attn_fwd2.cu -- K8 v2: causal attention forward on tcgen05 for prefill-chunk and finetuning-
// window rows (attention_rows, tiny_model.hpp:118-151, over paged KV), two query tiles per CTA.
//
// One 128-row query tile per CTA would feed every 64 KB K/V tile only 8.4 MFLOP (128 FLOP per L2
// byte -- at the tensor peak that is the whole L2 bandwidth); this kernel (the FA4 structure,
// re-derived for GQA-packed paged KV):
//   * CTA = 2 query tiles x 128 GQA-packed rows sharing every K/V tile (256 FLOP / L2 byte);
//   * TMEM (512 cols): S0 | S1 | O0 | O1; softmax writes P_i (bf16) back into the first 64
//     columns of S_i and the PV MMA reads its A operand straight from TMEM (tcgen05.mma
//     [d], [a_tmem], b_desc): no P round trip through shared memory;
//   * one softmax warpgroup per query tile, one thread per row (the full 128-key row in
//     registers: no cross-thread max/sum exchange), lazy O rescale (only when a row's max
//     grows by > 2^8) done by the softmax thread itself while PV_{j-1} is known complete;
//   * warp 0 TMA producer (K and V on separate 2-stage rings, 128-row boxes for contiguous
//     page runs, 16-row page boxes otherwise), warp 1 MMA issuer (S0, S1, PV0, PV1 per tile;
//     S_i(j+1) waits for PV_i(j) because P_i aliases S_i), warp 2 TMEM allocator;
//   * setmaxnreg: the producer warpgroup shrinks to 56 registers, the softmax warpgroups grow
//     to 224 (a 128-float row + its bf16 pack live in registers).
#include <atomic>
#include <cstdio>

#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"

namespace cs {

namespace {
constexpr float kLn2f = 0.6931471805599453f;
constexpr int D2 = 128;
constexpr int BM2 = 128;             // packed rows per query tile
constexpr int BN2 = 128;             // keys per KV tile
constexpr int HALF2 = 128 * 128;     // [128 rows][128 B] SW128 half-tile (16 KB)
constexpr int TILE2 = 2 * HALF2;     // [128 x 128] bf16 (32 KB)
constexpr int SM_Q = 0;              // 2 query tiles
constexpr int SM_K = SM_Q + 2 * TILE2;
constexpr int SM_V = SM_K + 2 * TILE2;
constexpr int SM_BAR = SM_V + 2 * TILE2;
constexpr int SM_TOTAL2 = SM_BAR + 256 + 1024;
constexpr float kRescale2 = 8.0f;    // log2 units

CS_DEV uint32_t sw_off(int r, int c) {  // 16-byte chunk c (0..15) of row r, K-major SW128 tile
  return (uint32_t)((c >> 3) * HALF2 + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// O (+)= A[tmem] * B[smem]: kind::f16, A operand (M x K bf16) read from TMEM
CS_DEV void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

CS_DEV void tmem_st_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// paged K (or V) tile of 128 keys into two SW128 halves
CS_DEV void load_tile2(const CUtensorMap* t16, const CUtensorMap* t128, uint64_t* bar, uint8_t* dst,
                       const int* pt, int page_off, int P, int k0, int k_end, int kvh) {
  const int pg0 = __ldg(pt + page_off + k0 / P);
  bool contig = true;
  for (int key = (k0 / P + 1) * P; key < k0 + BN2 && key < k_end; key += P)
    contig &= __ldg(pt + page_off + key / P) == pg0 + (key / P - k0 / P);
  if (contig) {
    const int row = pg0 * P + (k0 % P);
    for (int h = 0; h < 2; ++h) tma_load_2d(t128, bar, dst + h * HALF2, kvh * D2 + h * 64, row);
  } else {
    for (int ch = 0; ch < BN2 / 16; ++ch) {
      const int key0 = k0 + ch * 16;
      const int row = key0 < k_end ? __ldg(pt + page_off + key0 / P) * P + (key0 % P) : 0;
      for (int h = 0; h < 2; ++h)
        tma_load_2d(t16, bar, dst + h * HALF2 + ch * 2048, kvh * D2 + h * 64, row);
    }
  }
}
}  // namespace

__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmK128,
                        const __grid_constant__ CUtensorMap tmV128, AttnFwdParams p) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM_BAR);
  uint64_t* k_full = bars + 0;    // [2]
  uint64_t* k_empty = bars + 2;   // [2]
  uint64_t* v_full = bars + 4;    // [2]
  uint64_t* v_empty = bars + 6;   // [2]
  uint64_t* s_full = bars + 8;    // [2] per query tile
  uint64_t* p_full = bars + 10;   // [2] per query tile
  uint64_t* pv_done = bars + 12;  // [2] per query tile
  uint64_t* q_full = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const AttnWork w = p.work[blockIdx.x];
  const AttnSeg sg = p.segs[w.seg];
  const int grp = p.grp;
  const int rpt = BM2 / grp;  // query positions per tile
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;  // warp-uniform
  // keys [k_begin, k_end) of the item (k_begin a multiple of 128; > 0 for split-KV parts)
  const int j0 = w.k_begin / BN2;
  const int nt = (w.k_end + BN2 - 1) / BN2 - j0;
  const int ntile = w.nq > rpt ? 2 : 1;  // query tiles of this item (small calls use 1)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmK128);
    tma_prefetch_desc(&tmV128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(q_full, 256);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------ TMA producer
      for (int j = 0; j < nt; ++j) {
        const int st = j & 1, ph = ((j >> 1) & 1) ^ 1;
        mbar_wait(&k_empty[st], ph);
        mbar_arrive_expect_tx(&k_full[st], TILE2);
        load_tile2(&tmK, &tmK128, &k_full[st], smem + SM_K + st * TILE2, p.page_table, sg.page_off,
                   p.page_size, (j0 + j) * BN2, w.k_end, w.kv_head);
        mbar_wait(&v_empty[st], ph);
        mbar_arrive_expect_tx(&v_full[st], TILE2);
        load_tile2(&tmV, &tmV128, &v_full[st], smem + SM_V + st * TILE2, p.page_table, sg.page_off,
                   p.page_size, (j0 + j) * BN2, w.k_end, w.kv_head);
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------ MMA issuer
      // the whole warp walks the schedule (descriptors in uniform registers: no per-MMA
      // R2UR / elect loop), one elected lane issues each group of MMAs and its commit
      constexpr uint32_t idS = idesc_bf16_f32_major(128, 128, 0, 0);
      constexpr uint32_t idO = idesc_bf16_f32_major(128, 128, 0, 1);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto qk = [&](int i, uint32_t sK) {
        const uint32_t sQ = smem_u32(smem + SM_Q + i * TILE2);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D2 / 16; ++kk) {
            const uint64_t a = umma_desc_sw128(sQ + (kk >> 2) * HALF2 + (kk & 3) * 32);
            const uint64_t b = umma_desc_sw128(sK + (kk >> 2) * HALF2 + (kk & 3) * 32);
            mma_bf16(tmem + i * 128, a, b, idS, kk > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[i]);
        }
        __syncwarp();
      };
      auto pv = [&](int i, uint32_t sV, int j) {
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN2 / 16; ++kk) {
            const uint64_t b = umma_desc_sw128_mn(sV + kk * 2048, HALF2, 1024);
            mma_bf16_ts(tmem + 256 + i * 128, tmem + i * 128 + kk * 8, b, idO, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&pv_done[i]);
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) mma_commit(bar);
        __syncwarp();
      };
      if (ntile == 2) {
        // ping-pong: while the softmax of query tile 0 runs on S_0(j), the tensor pipe does
        // PV_1(j-1) and QK_1(j); while tile 1's softmax runs, PV_0(j) and QK_0(j+1)
        for (int j = 0; j < nt; ++j) {
          const int st = j & 1, pst = (j - 1) & 1;
          mbar_wait(&k_full[st], (j >> 1) & 1);
          if (j > 0) mbar_wait(&pv_done[0], (j - 1) & 1);  // P_0(j-1) (aliases S_0) consumed
          tc_fence_after();
          const uint32_t sK = smem_u32(smem + SM_K + st * TILE2);
          qk(0, sK);
          if (j > 0) {
            mbar_wait(&p_full[1], (j - 1) & 1);
            tc_fence_after();
            pv(1, smem_u32(smem + SM_V + pst * TILE2), j - 1);
            commit(&v_empty[pst]);  // V(j-1) fully consumed
            mbar_wait(&pv_done[1], (j - 1) & 1);
            tc_fence_after();
          }
          qk(1, sK);
          commit(&k_empty[st]);
          mbar_wait(&v_full[st], (j >> 1) & 1);
          mbar_wait(&p_full[0], j & 1);
          tc_fence_after();
          pv(0, smem_u32(smem + SM_V + st * TILE2), j);
        }
        if (nt > 0) {
          const int lst = (nt - 1) & 1;
          mbar_wait(&p_full[1], (nt - 1) & 1);
          tc_fence_after();
          pv(1, smem_u32(smem + SM_V + lst * TILE2), nt - 1);
          commit(&v_empty[lst]);
        }
      } else {
        for (int j = 0; j < nt; ++j) {
          const int st = j & 1;
          mbar_wait(&k_full[st], (j >> 1) & 1);
          if (j > 0) mbar_wait(&pv_done[0], (j - 1) & 1);  // P_0(j-1) aliases S_0
          tc_fence_after();
          qk(0, smem_u32(smem + SM_K + st * TILE2));
          commit(&k_empty[st]);
          mbar_wait(&v_full[st], (j >> 1) & 1);
          mbar_wait(&p_full[0], j & 1);
          tc_fence_after();
          pv(0, smem_u32(smem + SM_V + st * TILE2), j);
          commit(&v_empty[st]);
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ------------------------------------------------------------ softmax / epilogue
    const int qt = (warp - 4) >> 2;       // query tile of this warpgroup
    const int ew = warp & 3;              // TMEM lane quarter
    const int r = ew * 32 + lane;         // packed row in the tile == TMEM lane
    const int qr = qt * rpt + r / grp, gi = r % grp;
    const bool valid = (r / grp) < rpt && qr < w.nq;
    const int pos = valid ? sg.ctx_start + w.q0 + qr : -1;
    const int qh = w.kv_head * grp + gi;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const uint32_t tS = tmem + lane_base + qt * 128;
    const uint32_t tO = tmem + lane_base + 256 + qt * 128;
    {  // Q tile row (16 x 16B chunks, K-major SW128)
      uint8_t* sq = smem + SM_Q + qt * TILE2;
      const bf16* src = p.q + (long)(sg.q_start + w.q0 + (valid ? qr : 0)) * p.q_ld + (long)qh * D2;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (valid) v = *reinterpret_cast<const uint4*>(src + c * 8);
        *reinterpret_cast<uint4*>(sq + sw_off(r, c)) = v;
      }
      fence_proxy_async_smem();
      mbar_arrive(q_full);
    }
    float m_ref = -INFINITY, l_sum = 0.f;
    const int nt_me = qt < ntile ? nt : 0;
    for (int j = 0; j < nt_me; ++j) {
      mbar_wait(&s_full[qt], j & 1);
      tc_fence_after();
      float s[BN2];
      {
        uint32_t u[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tS + c * 32, u[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(u[c][i]);
      }
      // raw scores: max first (scale > 0), masking only on tiles that touch the diagonal /
      // k_end; then x = s * scale_log2 - m (FFMA2), 2^x on the SFU, row sums on FADD2
      const int kbase = (j0 + j) * BN2;
      if (!(kbase + BN2 - 1 <= pos && kbase + BN2 <= w.k_end)) {
#pragma unroll
        for (int i = 0; i < BN2; ++i)
          if (kbase + i > pos || kbase + i >= w.k_end) s[i] = -INFINITY;
      }
      float mr = -INFINITY;
#pragma unroll
      for (int i = 0; i < BN2; i += 2) mr = fmaxf(mr, fmaxf(s[i], s[i + 1]));
      const float mx = mr * p.scale_log2;
      bool rescale = false;
      float factor = 1.f;
      if (mx > m_ref + kRescale2 || (m_ref == -INFINITY && mx > -INFINITY)) {
        factor = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - mx);
        rescale = j > 0 && m_ref != -INFINITY;
        m_ref = mx;
        l_sum *= factor;
      }
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
      const float nb = m_ref == -INFINITY ? 0.f : -m_ref;
      const float2 nb2 = make_float2(nb, nb);
      float2 rs2 = make_float2(0.f, 0.f);
      // P (bf16) into the first 64 columns of S_i: every S column was read above
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float2 x = ffma2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nb2);
          x.x = ex2_approx(x.x);
          x.y = ex2_approx(x.y);
          rs2 = fadd2(rs2, x);
          pk[i] = pack_bf16(x.x, x.y);
        }
        tmem_st_x16(tS + c * 16, pk);
      }
      const float rs = rs2.x + rs2.y;
      l_sum += rs;
      // O rescale (warp-collective tcgen05.ld/st): PV_i(j-1) must be complete first
      if (__any_sync(0xffffffffu, rescale)) {
        mbar_wait(&pv_done[qt], (j - 1) & 1);
        tc_fence_after();
        if (!rescale) factor = 1.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(tO + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 v = fmul2(make_float2(__uint_as_float(o[i]), __uint_as_float(o[i + 1])),
                                   make_float2(factor, factor));
            o[i] = __float_as_uint(v.x);
            o[i + 1] = __float_as_uint(v.y);
          }
          tmem_st_32x32b_x32(tO + c * 32, o);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[qt]);
    }
    // epilogue: wait for the last PV of this tile, O / l, LSE (an unused tile has no rows)
    if (nt_me > 0) {
      mbar_wait(&pv_done[qt], (nt_me - 1) & 1);
      tc_fence_after();
    }
    const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
    const float lse_v = l_sum > 0.f ? (m_ref + __log2f(l_sum)) * kLn2f : -INFINITY;
    if (w.part >= 0) {
      // split-KV part: normalised O (fp32) and LSE, dense (position, head) rows of the item;
      // attn_combine_kernel (part_rows = 256) merges the parts
      const long prow = (long)w.part * 256 + (long)(qr * grp + gi);
      float* dst = p.part_o + prow * D2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tO + c * 32, o);
        tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + c * 32 + i) =
                make_float4(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv,
                            __uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
        }
      }
      if (valid) p.part_lse[prow] = lse_v;
    } else {
      bf16* dst = p.out + (long)(sg.q_start + w.q0 + (valid ? qr : 0)) * p.out_ld + (long)qh * D2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tO + c * 32, o);
        tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + c * 32 + i) = v;
          }
        }
      }
      if (valid && p.lse) p.lse[(long)(sg.q_start + w.q0 + qr) * p.lse_ld + qh] = lse_v;
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

cudaError_t attn_fwd_tc2(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                         const CUtensorMap& tmK128, const CUtensorMap& tmV128, int n_work,
                         cudaStream_t st) {
  if (n_work <= 0) return cudaSuccess;
  static bool once = (cudaFuncSetAttribute(attn_fwd_tc2_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, SM_TOTAL2),
                      true);
  (void)once;
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(attn_fwd_tc2_kernel, dim3(n_work), dim3(384), SM_TOTAL2, st, tmK, tmV, tmK128, tmV128, p);
  return cudaGetLastError();
}

}  // namespace cs
