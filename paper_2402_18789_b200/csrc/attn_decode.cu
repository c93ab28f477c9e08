// attn_decode.cu -- K7: paged-KV decode attention, the HBM-bound part of attention_rows
// (tiny_model.hpp:118-151) for decode rows (and any segment whose GQA-packed rows fit one
// m16 tile: q_len * group <= 16).
//
// Work item = (segment, kv head, key range [k_begin, k_end)); the host balances the key
// ranges over the SMs (flash-decoding split).  Every warp is a persistent stream over items:
//   * its own STAGES-deep TMA ring: lane 0 issues each 32-key tile as 16-row boxes (one page
//     chunk each, SWIZZLE_128B) for K and V on one mbarrier -- 8 instructions per 16 KB
//     instead of a per-lane page-table walk (the cp.async version spent most of its issue
//     slots on that address arithmetic; profiles/r1_decode_ncu.txt), running across items;
//   * attn_decode_swap_kernel (items of <= 8 GQA-packed rows, every decode row of LLaMA /
//     Qwen): swapped operands, S^T = K Q^T and O^T = V^T P^T on mma.sync with the keys / head
//     dims on M and the rows on N = 8;
//   * attn_decode_stream_kernel (9-16 rows): the rows on M = 16.
// Split items' partials are merged by attn_combine_kernel (PDL-launched).  Merging them in
// the decode kernel instead -- the part that finishes last reads the group's partials --
// measured slower at the 8B operating point (35.8 -> 52.6 us per launch: every part pays a
// threadfence + atomic, and the merging warp's dependent loads stall its stream).
// Online softmax in the log2 domain; only K/V bytes touch HBM in the loop: the algorithmic
// traffic is 2 * ctx * d * 2 B per (request, kv head).
#include <cfloat>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"
#include "mma.cuh"

namespace cs {

#ifdef CS_DEC_TRACE
// experiment build only: per-warp globaltimer stamps of the swap kernel (start, first tile
// landed, end, tiles, SM) -- scripts/decode_trace.py
__device__ unsigned long long* g_dec_trace = nullptr;
CS_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

namespace {
constexpr float kLn2 = 0.6931471805599453f;

template <int D, int KT>
constexpr int stage_bytes() {
  return 2 * KT * D * 2;  // K + V
}
template <int D, int KT, int NWARP, int STAGES>
constexpr int dec_smem() {
  return 1024 + NWARP * STAGES * stage_bytes<D, KT>() + NWARP * STAGES * 8;
}

CS_DEV uint32_t ld_u32(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const unsigned int*>(p)); }

// byte offset of 16-byte chunk c (0..D/8-1) of key row r in a [KT x D] bf16 tile that TMA
// wrote as D/64 column halves of [KT rows x 128 B] with SWIZZLE_128B
template <int KT>
CS_DEV uint32_t tile_off(int r, int c) {
  return (uint32_t)((c >> 3) * (KT * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}
}  // namespace

// ---------------------------------------------------------------- persistent streams
// Every warp is an independent, persistent stream over whole work items (items gw, gw + W,
// ... for W warps in the grid; the host sorts items longest first): no cross-warp merge, the
// item's normalised output (or split-KV partial + LSE) leaves straight from the mma
// fragments.  The warp's TMA ring runs ACROSS item boundaries -- while the last tiles of item
// i are in the tensor pipe, lane 0 already has item i+1's first tiles in flight -- so the
// per-item prologue (work load, first TMA round trip) and epilogue (stores) overlap the
// stream instead of idling the SM (the per-item CTA version spent ~40% of a bench-sized
// launch there: ncu long-scoreboard stalls on the work / page-table loads).
template <int D, int KT, int NWARP, int STAGES>
__global__ void __launch_bounds__(NWARP * 32, 1)
    attn_decode_stream_kernel(const __grid_constant__ CUtensorMap tmK,
                              const __grid_constant__ CUtensorMap tmV, AttnFwdParams p, int n_items) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  constexpr int NH = D / 64;
  constexpr int HALF = KT * 128;
  constexpr int TILE = NH * HALF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TW = gridDim.x * NWARP;
  const int gw = blockIdx.x * NWARP + warp;
  uint8_t* ws = smem + warp * (STAGES * 2 * TILE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NWARP * STAGES * 2 * TILE) + warp * STAGES;
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  __syncwarp();
  if (gw >= n_items) return;
  const int grp = p.grp;
  struct Item {
    int q_row, pos0, page_off, kv_head, k_begin, k_end, part, nq;
  };
  auto load_item = [&](int it) {
    const int4* q = reinterpret_cast<const int4*>(p.dwork + it);
    const int4 a = __ldg(q), b = __ldg(q + 1);
    return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  };
  // ---- issue side (lane 0): (item, tile) cursor running up to STAGES-1 tiles ahead
  int is_item = gw, is_t = 0, is_n = 0;  // item, next tile in it, tiles in it
  Item iw{};
  long g_issue = 0, g_cons = 0;
  auto issue_open = [&]() {
    iw = load_item(is_item);
    is_t = 0;
    is_n = (iw.k_end + KT - 1) / KT - iw.k_begin / KT;
  };
  auto top_up = [&]() {
    while (is_item < n_items && g_issue < g_cons + STAGES) {
      const int st = (int)(g_issue % STAGES);
      uint8_t* dk = ws + st * 2 * TILE;
      uint8_t* dv = dk + TILE;
      mbar_arrive_expect_tx(&full[st], 2 * TILE);
      const int kt = iw.k_begin / KT + is_t;
      const int last_box = (iw.k_end - 1) & ~15;
      const AttnDecWork* wp = p.dwork + is_item;
#pragma unroll
      for (int b = 0; b < KT / 16; ++b) {
        const int jb = min(kt * KT + b * 16, last_box);
        const int bi = (jb - iw.k_begin) >> 4;
        const int prow = bi < 8 ? __ldg(wp->prow + bi)
                                : __ldg(p.page_table + iw.page_off + jb / p.page_size) * p.page_size + jb % p.page_size;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          const int col = iw.kv_head * D + hh * 64;
          tma_load_2d(&tmK, &full[st], dk + hh * HALF + b * 2048, col, prow);
          tma_load_2d(&tmV, &full[st], dv + hh * HALF + b * 2048, col, prow);
        }
      }
      ++g_issue;
      if (++is_t == is_n) {
        is_item += TW;
        if (is_item < n_items) issue_open();
      }
    }
  };
  if (lane == 0) {
    issue_open();
    top_up();
  }
  const int ra = lane >> 2, rb = ra + 8;
  for (int item = gw; item < n_items; item += TW) {
    const Item w = load_item(item);
    const int nrows = w.nq * grp;
    const __nv_bfloat16* qa = nullptr;
    const __nv_bfloat16* qb = nullptr;
    if (ra < nrows) qa = p.q + (long)(w.q_row + ra / grp) * p.q_ld + (long)(w.kv_head * grp + ra % grp) * D;
    if (rb < nrows) qb = p.q + (long)(w.q_row + rb / grp) * p.q_ld + (long)(w.kv_head * grp + rb % grp) * D;
    uint32_t qf[D / 16][4];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int col = kk * 16 + 2 * (lane & 3);
      qf[kk][0] = qa ? ld_u32(qa + col) : 0u;
      qf[kk][1] = qb ? ld_u32(qb + col) : 0u;
      qf[kk][2] = qa ? ld_u32(qa + col + 8) : 0u;
      qf[kk][3] = qb ? ld_u32(qb + col + 8) : 0u;
    }
    const int pos_a = ra < nrows ? w.pos0 + ra / grp : -1;
    const int pos_b = rb < nrows ? w.pos0 + rb / grp : -1;
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
    const int kt0 = w.k_begin / KT, nt = (w.k_end + KT - 1) / KT - kt0;
    for (int t = 0; t < nt; ++t) {
      if (lane == 0) top_up();
      const int st = (int)(g_cons % STAGES);
      mbar_wait(&full[st], (uint32_t)((g_cons / STAGES) & 1));
      const uint32_t kb = smem_u32(ws + st * 2 * TILE), vb = kb + TILE;
      const int kt = kt0 + t;
      float s[KT / 8][4];
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int nbp = 0; nbp < KT / 16; ++nbp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + tile_off<KT>(nbp * 16 + (lane & 7) + ((lane >> 4) << 3), kk * 2 + ((lane >> 3) & 1)),
                  b0, b1, b2, b3);
          mma16816(s[2 * nbp], qf[kk], b0, b1);
          mma16816(s[2 * nbp + 1], qf[kk], b2, b3);
        }
      }
      float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
      for (int nb = 0; nb < KT / 8; ++nb) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = kt * KT + nb * 8 + 2 * (lane & 3) + (e & 1);
          const int pos = e < 2 ? pos_a : pos_b;
          float v = s[nb][e] * p.scale_log2;
          if (j > pos || j >= w.k_end) v = -INFINITY;
          s[nb][e] = v;
        }
        mx_a = fmaxf(mx_a, fmaxf(s[nb][0], s[nb][1]));
        mx_b = fmaxf(mx_b, fmaxf(s[nb][2], s[nb][3]));
      }
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
      const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
      const float mu_a = mn_a == -INFINITY ? 0.f : mn_a;
      const float mu_b = mn_b == -INFINITY ? 0.f : mn_b;
      float rs_a = 0.f, rs_b = 0.f;
#pragma unroll
      for (int nb = 0; nb < KT / 8; ++nb) {
        s[nb][0] = exp2f(s[nb][0] - mu_a);
        s[nb][1] = exp2f(s[nb][1] - mu_a);
        s[nb][2] = exp2f(s[nb][2] - mu_b);
        s[nb][3] = exp2f(s[nb][3] - mu_b);
        rs_a += s[nb][0] + s[nb][1];
        rs_b += s[nb][2] + s[nb][3];
      }
      if (__any_sync(0xffffffffu, mn_a != m_a || mn_b != m_b)) {
        const float c_a = exp2f(m_a - mu_a), c_b = exp2f(m_b - mu_b);
        l_a *= c_a;
        l_b *= c_b;
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          o[n][0] *= c_a;
          o[n][1] *= c_a;
          o[n][2] *= c_b;
          o[n][3] *= c_b;
        }
      }
      m_a = mn_a;
      m_b = mn_b;
      l_a += rs_a;
      l_b += rs_b;
#pragma unroll
      for (int kk = 0; kk < KT / 16; ++kk) {
        uint32_t a[4];
        a[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
        a[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
        a[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
        a[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
        for (int dp = 0; dp < D / 16; ++dp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + tile_off<KT>(kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), dp * 2 + (lane >> 4)),
                    b0, b1, b2, b3);
          mma16816(o[2 * dp], a, b0, b1);
          mma16816(o[2 * dp + 1], a, b2, b3);
        }
      }
      __syncwarp();  // every lane is done reading this stage before lane 0 refills it
      ++g_cons;
    }
    // ---- epilogue straight from the fragments (the next item's tiles are already in flight)
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int r = half ? rb : ra;
      if (r >= nrows) continue;
      const float L = half ? l_b : l_a, M = half ? m_b : m_a;
      const float inv = L > 0.f ? 1.f / L : 0.f;
      const float lse = L > 0.f ? (M + __log2f(L)) * kLn2 : -INFINITY;
      const int qr = r / grp, g = r - qr * grp;
      if (w.part < 0) {
        const long row = w.q_row + qr;
        const int qh = w.kv_head * grp + g;
        __nv_bfloat16* dst = p.out + row * p.out_ld + (long)qh * D;
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          const int d = n * 8 + 2 * (lane & 3);
          *reinterpret_cast<uint32_t*>(dst + d) = pack_bf16(o[n][2 * half] * inv, o[n][2 * half + 1] * inv);
        }
        if ((lane & 3) == 0 && p.lse) p.lse[row * p.lse_ld + qh] = lse;
      } else {
        float* dst = p.part_o + ((long)w.part * 64 + r) * D;
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          const int d = n * 8 + 2 * (lane & 3);
          *reinterpret_cast<float2*>(dst + d) = make_float2(o[n][2 * half] * inv, o[n][2 * half + 1] * inv);
        }
        if ((lane & 3) == 0) p.part_lse[(long)w.part * 64 + r] = lse;
      }
    }
  }
}

// ---------------------------------------------------------------- swapped operands
// Decode rows are the GQA group of ONE query position (4 rows for LLaMA-8B, 5 for Qwen): the
// kernels above put them on the M=16 side of mma.m16n8k16 and waste 3/4 of every MMA.  Here the
// keys and head dims take the M side and the (<= 8) packed query rows the N=8 side:
//   S^T[32 keys x 8 rows] = K . Q^T   (A = K tile via ldmatrix, B = Q^T fragments in registers)
//   O^T[128 d x 8 rows]  += V^T . P^T (A = V^T via ldmatrix.trans, B = P^T)
// P^T's accumulator fragment (key rows, query columns) becomes the B fragment (query rows,
// key columns) with one movmatrix.trans per 8x8 block.  Half the MMAs and half the exp2 per
// K/V byte of the M=16 formulation; the per-query softmax statistics are column reductions
// (shuffles across the 8 lanes that share a column pair).  Persistent per-warp streams over
// whole items with the TMA ring running across item boundaries, as above.
CS_DEV uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int D, int KT, int NWARP, int STAGES>
__global__ void __launch_bounds__(NWARP * 32, 1)
    attn_decode_swap_kernel(const __grid_constant__ CUtensorMap tmK,
                            const __grid_constant__ CUtensorMap tmV, AttnFwdParams p, int n_items) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  constexpr int NH = D / 64;
  constexpr int HALF = KT * 128;
  constexpr int TILE = NH * HALF;
  constexpr int MT = KT / 16;  // 16-key m-tiles of S^T (= k-steps of the PV product)
  constexpr int DM = D / 16;   // 16-dim m-tiles of O^T
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TW = gridDim.x * NWARP;
  const int gw = blockIdx.x * NWARP + warp;
  uint8_t* ws = smem + warp * (STAGES * 2 * TILE);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NWARP * STAGES * 2 * TILE) + warp * STAGES;
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  __syncwarp();
#ifdef CS_DEC_TRACE
  const unsigned long long tr_t0 = gtimer();
  unsigned long long tr_t1 = 0;
#endif
  if (gw >= n_items) return;
  const int grp = p.grp;
  struct Item {
    int q_row, pos0, page_off, kv_head, k_begin, k_end, part, nq;
  };
  auto load_item = [&](int it) {
    const int4* q = reinterpret_cast<const int4*>(p.dwork + it);
    const int4 a = __ldg(q), b = __ldg(q + 1);
    return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  };
  int is_item = gw, is_t = 0, is_n = 0;
  Item iw{};
  long g_issue = 0, g_cons = 0;
  auto issue_open = [&]() {
    iw = load_item(is_item);
    is_t = 0;
    is_n = (iw.k_end + KT - 1) / KT - iw.k_begin / KT;
  };
  auto top_up = [&]() {
    while (is_item < n_items && g_issue < g_cons + STAGES) {
      const int st = (int)(g_issue % STAGES);
      uint8_t* dk = ws + st * 2 * TILE;
      uint8_t* dv = dk + TILE;
      mbar_arrive_expect_tx(&full[st], 2 * TILE);
      const int kt = iw.k_begin / KT + is_t;
      const int last_box = (iw.k_end - 1) & ~15;
      const AttnDecWork* wp = p.dwork + is_item;
#pragma unroll
      for (int b = 0; b < KT / 16; ++b) {
        const int jb = min(kt * KT + b * 16, last_box);
        const int bi = (jb - iw.k_begin) >> 4;
        const int prow = bi < 8 ? __ldg(wp->prow + bi)
                                : __ldg(p.page_table + iw.page_off + jb / p.page_size) * p.page_size + jb % p.page_size;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          const int col = iw.kv_head * D + hh * 64;
          tma_load_2d(&tmK, &full[st], dk + hh * HALF + b * 2048, col, prow);
          tma_load_2d(&tmV, &full[st], dv + hh * HALF + b * 2048, col, prow);
        }
      }
      ++g_issue;
      if (++is_t == is_n) {
        is_item += TW;
        if (is_item < n_items) issue_open();
      }
    }
  };
  if (lane == 0) {
    issue_open();
    top_up();
  }
  const int g = lane >> 2, t = lane & 3;
  for (int item = gw; item < n_items; item += TW) {
    const Item w = load_item(item);
    const int nrows = w.nq * grp;  // <= 8
    // B fragments of Q^T: lane holds Q[row g][d = 16 kk + 2t (+8), +1]
    uint32_t qf[D / 16][2];
    {
      const __nv_bfloat16* qr = g < nrows
                                    ? p.q + (long)(w.q_row + g / grp) * p.q_ld + (long)(w.kv_head * grp + g % grp) * D
                                    : nullptr;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        qf[kk][0] = qr ? ld_u32(qr + kk * 16 + 2 * t) : 0u;
        qf[kk][1] = qr ? ld_u32(qr + kk * 16 + 8 + 2 * t) : 0u;
      }
    }
    // this lane's two query columns 2t, 2t+1
    const int c0 = 2 * t, c1 = 2 * t + 1;
    const int pos_0 = c0 < nrows ? w.pos0 + c0 / grp : -1;
    const int pos_1 = c1 < nrows ? w.pos0 + c1 / grp : -1;
    float o[DM][4];
#pragma unroll
    for (int i = 0; i < DM; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_0 = -INFINITY, m_1 = -INFINITY, l_0 = 0.f, l_1 = 0.f;
    const int kt0 = w.k_begin / KT, nt = (w.k_end + KT - 1) / KT - kt0;
    for (int tt = 0; tt < nt; ++tt) {
      if (lane == 0) top_up();
      const int st = (int)(g_cons % STAGES);
      mbar_wait(&full[st], (uint32_t)((g_cons / STAGES) & 1));
#ifdef CS_DEC_TRACE
      if (g_cons == 0) tr_t1 = gtimer();
#endif
      const uint32_t kb = smem_u32(ws + st * 2 * TILE), vb = kb + TILE;
      const int kt = kt0 + tt;
      // ---- S^T = K Q^T
      float s[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) s[mt][0] = s[mt][1] = s[mt][2] = s[mt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t a[4];
          ldsm_x4(kb + tile_off<KT>(mt * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), kk * 2 + (lane >> 4)),
                  a[0], a[1], a[2], a[3]);
          mma16816(s[mt], a, qf[kk][0], qf[kk][1]);
        }
      }
      // ---- mask + column (per query) online softmax
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = kt * KT + mt * 16 + g + ((e >> 1) << 3);
          const int pos = (e & 1) ? pos_1 : pos_0;
          float v = s[mt][e] * p.scale_log2;
          if (j > pos || j >= w.k_end) v = -INFINITY;
          s[mt][e] = v;
        }
        mx0 = fmaxf(mx0, fmaxf(s[mt][0], s[mt][2]));
        mx1 = fmaxf(mx1, fmaxf(s[mt][1], s[mt][3]));
      }
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, x));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, x));
      }
      const float mn0 = fmaxf(m_0, mx0), mn1 = fmaxf(m_1, mx1);
      const float mu0 = mn0 == -INFINITY ? 0.f : mn0;
      const float mu1 = mn1 == -INFINITY ? 0.f : mn1;
      float rs0 = 0.f, rs1 = 0.f;
      uint32_t pb[MT][2];  // P^T as B fragments of the PV product
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const float p0 = ex2_approx(s[mt][0] - mu0), p1 = ex2_approx(s[mt][1] - mu1);
        const float p2 = ex2_approx(s[mt][2] - mu0), p3 = ex2_approx(s[mt][3] - mu1);
        rs0 += p0 + p2;
        rs1 += p1 + p3;
        pb[mt][0] = movmatrix_t(pack_bf16(p0, p1));  // keys 16mt + 0..7
        pb[mt][1] = movmatrix_t(pack_bf16(p2, p3));  // keys 16mt + 8..15
      }
      if (__any_sync(0xffffffffu, mn0 != m_0 || mn1 != m_1)) {
        const float f0 = ex2_approx(m_0 - mu0), f1 = ex2_approx(m_1 - mu1);
        l_0 *= f0;
        l_1 *= f1;
#pragma unroll
        for (int i = 0; i < DM; ++i) {
          o[i][0] *= f0;
          o[i][1] *= f1;
          o[i][2] *= f0;
          o[i][3] *= f1;
        }
      }
      m_0 = mn0;
      m_1 = mn1;
      l_0 += rs0;
      l_1 += rs1;
      // ---- O^T += V^T P^T
#pragma unroll
      for (int ks = 0; ks < MT; ++ks) {
#pragma unroll
        for (int dm = 0; dm < DM; ++dm) {
          uint32_t a[4];
          ldsm_x4_t(vb + tile_off<KT>(ks * 16 + (lane & 7) + ((lane >> 4) << 3), dm * 2 + ((lane >> 3) & 1)),
                    a[0], a[1], a[2], a[3]);
          mma16816(o[dm], a, pb[ks][0], pb[ks][1]);
        }
      }
      __syncwarp();  // every lane is done reading this stage before lane 0 refills it
      ++g_cons;
    }
    // ---- epilogue: column sums, normalise, store O[q][d] (the next item's tiles are in flight)
#pragma unroll
    for (int x = 4; x < 32; x <<= 1) {
      l_0 += __shfl_xor_sync(0xffffffffu, l_0, x);
      l_1 += __shfl_xor_sync(0xffffffffu, l_1, x);
    }
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int q = cc ? c1 : c0;
      if (q >= nrows) continue;
      const float L = cc ? l_1 : l_0, M = cc ? m_1 : m_0;
      const float inv = L > 0.f ? 1.f / L : 0.f;
      const int qr = q / grp, hq = w.kv_head * grp + (q - qr * grp);
      if (w.part < 0) {
        const long row = w.q_row + qr;
        __nv_bfloat16* dst = p.out + row * p.out_ld + (long)hq * D;
#pragma unroll
        for (int dm = 0; dm < DM; ++dm) {
          dst[dm * 16 + g] = __float2bfloat16(o[dm][cc] * inv);
          dst[dm * 16 + g + 8] = __float2bfloat16(o[dm][2 + cc] * inv);
        }
        if (g == 0 && p.lse) p.lse[row * p.lse_ld + hq] = L > 0.f ? (M + __log2f(L)) * kLn2 : -INFINITY;
      } else {
        float* dst = p.part_o + ((long)w.part * 64 + q) * D;
#pragma unroll
        for (int dm = 0; dm < DM; ++dm) {
          dst[dm * 16 + g] = o[dm][cc] * inv;
          dst[dm * 16 + g + 8] = o[dm][2 + cc] * inv;
        }
        if (g == 0) p.part_lse[(long)w.part * 64 + q] = L > 0.f ? (M + __log2f(L)) * kLn2 : -INFINITY;
      }
    }
  }
#ifdef CS_DEC_TRACE
  if (lane == 0 && g_dec_trace) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* o = g_dec_trace + (long)gw * 5;
    o[0] = tr_t0; o[1] = tr_t1; o[2] = gtimer(); o[3] = (unsigned long long)g_cons; o[4] = smid;
  }
#endif
}

namespace {
template <int D, int KT, int NW, int ST>
cudaError_t launch_dec_swap(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                            int n_work, cudaStream_t st) {
  constexpr int smem = dec_smem<D, KT, NW, ST>();
  static bool once = (cudaFuncSetAttribute(attn_decode_swap_kernel<D, KT, NW, ST>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                      true);
  (void)once;
  const int cps = std::max(1, std::min(16, (228 * 1024) / (smem + 1024)));
  const int grid = std::max(1, std::min((n_work + NW - 1) / NW, 148 * cps));
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(attn_decode_swap_kernel<D, KT, NW, ST>, dim3(grid), dim3(NW * 32), smem, st, tmK, tmV, p, n_work);
  return cudaGetLastError();
}

template <int D, int KT, int NW, int ST>
cudaError_t launch_dec_stream(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                              int n_work, cudaStream_t st) {
  constexpr int smem = dec_smem<D, KT, NW, ST>();
  static bool once = (cudaFuncSetAttribute(attn_decode_stream_kernel<D, KT, NW, ST>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                      true);
  (void)once;
  const int cps = std::max(1, std::min(16, (228 * 1024) / (smem + 1024)));
  const int grid = std::max(1, std::min((n_work + NW - 1) / NW, 148 * cps));
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(attn_decode_stream_kernel<D, KT, NW, ST>, dim3(grid), dim3(NW * 32), smem, st, tmK, tmV, p, n_work);
  return cudaGetLastError();
}

// 32-key tiles, 2 warps x 2 stages per CTA, 3 CTAs per SM (scripts/decode_op.py: of the
// {32, 16}-key x {2, 4}-warp x {2, 3, 4}-stage variants this is the fastest at the bench's
// operating point, 100 rows x ~400 keys: 0.71 of measured HBM for the kernel)
#ifndef CS_DEC_NW
#define CS_DEC_NW 2
#endif
#ifndef CS_DEC_ST
#define CS_DEC_ST 2
#endif
constexpr int kDecKT = 32, kDecNW = CS_DEC_NW, kDecST = CS_DEC_ST;

template <int D>
cudaError_t launch_dec_d(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                         int n_work, cudaStream_t st) {
  if (p.max_dec_rows <= 8) return launch_dec_swap<D, kDecKT, kDecNW, kDecST>(p, tmK, tmV, n_work, st);
  return launch_dec_stream<D, kDecKT, kDecNW, kDecST>(p, tmK, tmV, n_work, st);
}
}  // namespace

void attn_decode_geometry(int head_dim, int* keys_per_tile, int* nwarp, int* ctas_per_sm,
                          int* streams) {
  const int smem = 1024 + kDecNW * kDecST * 2 * kDecKT * head_dim * 2 + kDecNW * kDecST * 8;
  *keys_per_tile = kDecKT;
  *nwarp = kDecNW;
  *ctas_per_sm = std::max(1, std::min(16, (228 * 1024) / (smem + 1024)));
  *streams = 2;
}

cudaError_t attn_decode(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                        int head_dim, int n_work, cudaStream_t st) {
  if (n_work <= 0) return cudaSuccess;
  if (head_dim == 128) return launch_dec_d<128>(p, tmK, tmV, n_work, st);
  if (head_dim == 64) return launch_dec_d<64>(p, tmK, tmV, n_work, st);
  return cudaErrorInvalidValue;
}

}  // namespace cs

#ifdef CS_DEC_TRACE
extern "C" int cs_debug_dec_trace(void* dev_buf) {
  return (int)cudaMemcpyToSymbol(cs::g_dec_trace, &dev_buf, sizeof(void*));
}
#endif
