// attn_tc.cu -- K8: causal attention forward on tcgen05 / TMEM for prefill-chunk and
// finetuning-window tiles (the compute-bound part of attention_rows, tiny_model.hpp:118-151,
// over paged KV).  Decode rows stay on the bandwidth kernel in attention.cu.
//
// CTA = 128 GQA-packed query rows ((q row, head-in-group) pairs sharing one KV head) x 1 KV
// head; loops over 128-key tiles up to the tile's last causal position.
//   warp 0     : TMA producer -- K and V tiles from the paged pools, one 16-key box per page
//                chunk and 64-column half (SWIZZLE_128B), 2-stage ring
//   warp 1     : MMA issuer  -- S_j = Q K_j^T (M=128,N=128,K=128) into one of two TMEM S
//                buffers; O += P_{j-1} V_{j-1} (V consumed MN-major straight from the
//                TMA tile: no transpose)
//   warp 2     : TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4..7 : softmax, one thread per query row (no shuffles): tcgen05.ld of the S row,
//                online max/sum in the log2 domain, lazy O rescale (only when the running
//                max grows by > 8, via tcgen05.ld/st on O), P written bf16 into a K-major
//                SWIZZLE_128B tile; epilogue O / l and the natural-log LSE.
#include <atomic>
#include <cstdio>

#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"

namespace cs {

namespace {
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int D = 128;          // head_dim
constexpr int BM = 128;         // packed query rows per CTA
constexpr int BN = 128;         // keys per tile
constexpr int HALF = BM * 128;  // one 64-column SW128 half of a [128 x 128] bf16 tile (16 KB)
constexpr int TILE = 2 * HALF;  // 32 KB
constexpr int SMEM_Q = 0;
constexpr int SMEM_P = SMEM_Q + TILE;
constexpr int SMEM_K = SMEM_P + TILE;        // 2 stages
constexpr int SMEM_V = SMEM_K + 2 * TILE;    // 2 stages
constexpr int SMEM_BAR = SMEM_V + 2 * TILE;  // barriers
constexpr int SMEM_TOTAL = SMEM_BAR + 128 + 4 * 768 + 1024;  // barriers + row exchange
constexpr float kRescaleThresh = 8.0f;  // log2 units

#ifdef CS_ATTN_DEBUG
CS_DEV void mbar_wait_dbg(uint64_t* bar, uint32_t phase, int tag, int j) {
  uint32_t ok = 0;
  const long lim = tag >= 6 ? (1L << 20) : (1L << 24);
  for (long it = 0; it < lim && !ok; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
  if (!ok) {
    printf("HANG blk %d thr %d tag %d j %d phase %u\n", blockIdx.x, threadIdx.x, tag, j, phase);
    __trap();
  }
}
#define MBW(b, ph, tag, j) mbar_wait_dbg(b, ph, tag, j)
#else
#define MBW(b, ph, tag, j) mbar_wait(b, ph)
#endif

// byte offset of 16-byte chunk c (0..15) of row r in a K-major SW128 [128 x 128] bf16 tile
CS_DEV uint32_t sw128_off(int r, int c) {
  return (uint32_t)((c >> 3) * HALF + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4));
}
}  // namespace

__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ CUtensorMap tmK128,
                       const __grid_constant__ CUtensorMap tmV128, AttnFwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
  uint64_t* kv_full = bars + 0;   // [2]
  uint64_t* kv_empty = bars + 2;  // [2]
  uint64_t* s_full = bars + 4;    // [2]
  uint64_t* s_free = bars + 6;    // [2]
  uint64_t* p_full = bars + 8;
  uint64_t* p_empty = bars + 9;   // PV_j complete (also: O safe to touch)
  uint64_t* q_full = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const AttnWork w = p.work[blockIdx.x];
  const AttnSeg sg = p.segs[w.seg];
  const int grp = p.grp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (w.k_end + BN - 1) / BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmK128);
    tma_prefetch_desc(&tmV128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 256);
    }
    mbar_init(p_full, 256);
    mbar_init(p_empty, 1);
    mbar_init(q_full, 256);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const int P = p.page_size;
      for (int j = 0; j < nt; ++j) {
        const int st = j & 1;
        MBW(&kv_empty[st], ((j >> 1) & 1) ^ 1, 1, j);
        mbar_arrive_expect_tx(&kv_full[st], 2 * TILE);
        uint8_t* sk = smem + SMEM_K + st * TILE;
        uint8_t* sv = smem + SMEM_V + st * TILE;
        // one 128-row box per half when the tile's pages are consecutive in the pool (the
        // finetuning sequence's pages are reserved as one run); else one box per 16 keys
        const int k0 = j * BN;
        const int pg0 = __ldg(p.page_table + sg.page_off + k0 / P);
        bool contig = true;
        for (int key = (k0 / P + 1) * P; key < k0 + BN && key < w.k_end; key += P)
          contig &= __ldg(p.page_table + sg.page_off + key / P) == pg0 + (key / P - k0 / P);
        if (contig) {
          const int row = pg0 * P + (k0 % P);
          for (int h = 0; h < 2; ++h) {
            const int col = w.kv_head * D + h * 64;
            tma_load_2d(&tmK128, &kv_full[st], sk + h * HALF, col, row);
            tma_load_2d(&tmV128, &kv_full[st], sv + h * HALF, col, row);
          }
        } else {
          for (int ch = 0; ch < BN / 16; ++ch) {
            const int key0 = k0 + ch * 16;
            int row = 0;
            if (key0 < w.k_end)
              row = __ldg(p.page_table + sg.page_off + key0 / P) * P + (key0 % P);
            for (int h = 0; h < 2; ++h) {
              const int col = w.kv_head * D + h * 64;
              tma_load_2d(&tmK, &kv_full[st], sk + h * HALF + ch * 16 * 128, col, row);
              tma_load_2d(&tmV, &kv_full[st], sv + h * HALF + ch * 16 * 128, col, row);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32_major(128, 128, 0, 0);
      constexpr uint32_t idO = idesc_bf16_f32_major(128, 128, 0, 1);
      const uint32_t sQ = smem_u32(smem + SMEM_Q), sP = smem_u32(smem + SMEM_P);
      const uint32_t tO = tmem + 256;
      MBW(q_full, 0, 2, 0);
      tc_fence_after();
      auto issue_pv = [&](int jj) {
        const int st = jj & 1;
        MBW(p_full, jj & 1, 3, jj);
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + SMEM_V + st * TILE);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t a = umma_desc_sw128(sP + (kk >> 2) * HALF + (kk & 3) * 32);
          const uint64_t b = umma_desc_sw128_mn(sV + kk * 2048, HALF, 1024);
          mma_bf16(tO, a, b, idO, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&kv_empty[st]);
        mma_commit(p_empty);
      };
      for (int j = 0; j < nt; ++j) {
        const int st = j & 1, sb = j & 1;
        MBW(&kv_full[st], (j >> 1) & 1, 4, j);
        MBW(&s_free[sb], ((j >> 1) & 1) ^ 1, 5, j);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + SMEM_K + st * TILE);
        const uint32_t tS = tmem + sb * 128;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t a = umma_desc_sw128(sQ + (kk >> 2) * HALF + (kk & 3) * 32);
          const uint64_t b = umma_desc_sw128(sK + (kk >> 2) * HALF + (kk & 3) * 32);
          mma_bf16(tS, a, b, idS, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[sb]);
        if (j > 0) issue_pv(j - 1);
      }
      if (nt > 0) issue_pv(nt - 1);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    // 8 warps: warp 4+ew (h=0) and 8+ew (h=1) share TMEM lanes [32ew, 32ew+32) = query rows;
    // h selects the 64-column half of S (and of O) each thread owns.
    const int ew = (warp - 4) & 3, hh = (warp - 4) >> 2;
    const int r = ew * 32 + lane;  // packed row == TMEM lane
    const int qr = r / grp, g = r % grp;
    const bool valid = qr < w.nq;
    const int pos = valid ? sg.ctx_start + w.q0 + qr : -1;
    const int qh = w.kv_head * grp + g;
    float* xch = reinterpret_cast<float*>(bars + 16);  // [2][2][128] partial row max / sum
    {  // Q tile: this thread's half row, 8 x 16B chunks, K-major SW128
      uint8_t* sq = smem + SMEM_Q;
      const bf16* src = p.q + (long)(sg.q_start + w.q0 + (valid ? qr : 0)) * p.q_ld + (long)qh * D;
#pragma unroll
      for (int c = hh * 8; c < hh * 8 + 8; ++c) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (valid) v = *reinterpret_cast<const uint4*>(src + c * 8);
        *reinterpret_cast<uint4*>(sq + sw128_off(r, c)) = v;
      }
      fence_proxy_async_smem();
      mbar_arrive(q_full);
    }
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    float m_ref = -INFINITY, l_sum = 0.f;
    uint8_t* sp = smem + SMEM_P;
    constexpr int HC = BN / 2;  // columns per thread
    for (int j = 0; j < nt; ++j) {
      const int sb = j & 1;
      MBW(&s_full[sb], (j >> 1) & 1, 6, j);
      tc_fence_after();
      float s[HC];
      {
        uint32_t r0[32], r1[32];
        tmem_ld_32x32b_x32(tmem + lane_base + sb * 128 + hh * HC, r0);
        tmem_ld_32x32b_x32(tmem + lane_base + sb * 128 + hh * HC + 32, r1);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = __uint_as_float(r0[i]);
          s[32 + i] = __uint_as_float(r1[i]);
        }
      }
      tc_fence_before();
      mbar_arrive(&s_free[sb]);
      // scale + causal mask (only tiles touching the diagonal / k_end), partial row max
      const int kbase = j * BN + hh * HC;
      float mx = -INFINITY;
      if (kbase + HC - 1 <= pos && kbase + HC <= w.k_end) {
#pragma unroll
        for (int i = 0; i < HC; ++i) {
          s[i] *= p.scale_log2;
          mx = fmaxf(mx, s[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < HC; ++i) {
          const int key = kbase + i;
          float v = s[i] * p.scale_log2;
          if (key > pos || key >= w.k_end) v = -INFINITY;
          s[i] = v;
          mx = fmaxf(mx, v);
        }
      }
      // exchange partial maxima between the two halves of the row
      float* slot = xch + (j & 1) * 256;
      slot[hh * 128 + r] = mx;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mx = fmaxf(mx, slot[(hh ^ 1) * 128 + r]);
      bool rescale = false;
      float factor = 1.f;
      if (mx > m_ref + kRescaleThresh || (m_ref == -INFINITY && mx > -INFINITY)) {
        factor = (m_ref == -INFINITY) ? 0.f : exp2f(m_ref - mx);
        rescale = j > 0 && m_ref != -INFINITY;
        m_ref = mx;
        l_sum *= factor;
      }
      const float base = m_ref == -INFINITY ? 0.f : m_ref;
      float rs = 0.f;
      uint32_t pk[HC / 2];
#pragma unroll
      for (int i = 0; i < HC; i += 2) {
        const float a = exp2f(s[i] - base), b = exp2f(s[i + 1] - base);
        rs += a + b;
        pk[i / 2] = pack_bf16(a, b);
      }
      l_sum += rs;
      // P buffer and O are free once PV_{j-1} completed
      if (j > 0) {
        MBW(p_empty, (j - 1) & 1, 7, j);
        tc_fence_after();
      }
      // tcgen05.ld/st are warp-collective (.sync.aligned): rescale as a warp when any row needs it
      if (__any_sync(0xffffffffu, rescale)) {
        if (!rescale) factor = 1.f;
        uint32_t o0[32], o1[32];
        const uint32_t ta = tmem + lane_base + 256 + hh * HC;
        tmem_ld_32x32b_x32(ta, o0);
        tmem_ld_32x32b_x32(ta + 32, o1);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          o0[i] = __float_as_uint(__uint_as_float(o0[i]) * factor);
          o1[i] = __float_as_uint(__uint_as_float(o1[i]) * factor);
        }
        tmem_st_32x32b_x32(ta, o0);
        tmem_st_32x32b_x32(ta + 32, o1);
        tmem_st_wait();
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(sp + sw128_off(r, hh * 8 + c)) =
            make_uint4(pk[c * 4], pk[c * 4 + 1], pk[c * 4 + 2], pk[c * 4 + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: total row sum across the halves, wait for the last PV, O / l, LSE
    xch[512 + hh * 128 + r] = l_sum;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    l_sum += xch[512 + (hh ^ 1) * 128 + r];
    if (nt > 0) {
      MBW(p_empty, (nt - 1) & 1, 8, nt);
      tc_fence_after();
    }
    const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
    bf16* dst = p.out + (long)(sg.q_start + w.q0 + (valid ? qr : 0)) * p.out_ld + (long)qh * D + hh * HC;
    {
      uint32_t o[2][32];
      tmem_ld_32x32b_x32(tmem + lane_base + 256 + hh * HC, o[0]);
      tmem_ld_32x32b_x32(tmem + lane_base + 256 + hh * HC + 32, o[1]);
      tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[c][i]) * inv, __uint_as_float(o[c][i + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(o[c][i + 2]) * inv, __uint_as_float(o[c][i + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(o[c][i + 4]) * inv, __uint_as_float(o[c][i + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(o[c][i + 6]) * inv, __uint_as_float(o[c][i + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + c * 32 + i) = v;
          }
      }
    }
    if (valid && hh == 0 && p.lse)
      p.lse[(long)(sg.q_start + w.q0 + qr) * p.lse_ld + qh] =
          l_sum > 0.f ? (m_ref + __log2f(l_sum)) * kLn2 : -INFINITY;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

cudaError_t attn_fwd_tc(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                        const CUtensorMap& tmK128, const CUtensorMap& tmV128, int n_work,
                        cudaStream_t st) {
  if (n_work <= 0) return cudaSuccess;
  static bool once = (cudaFuncSetAttribute(attn_fwd_tc_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           SMEM_TOTAL),
                      true);
  (void)once;
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  attn_fwd_tc_kernel<<<n_work, 384, SMEM_TOTAL, st>>>(tmK, tmV, tmK128, tmV128, p);
  return cudaGetLastError();
}

}  // namespace cs
