// attention.cu -- K7/K8/K9: causal attention over paged KV for the co-serving step.
//
// Forward (attn_fwd_kernel): replaces numdetail::attention_rows (tiny_model.hpp:118-151) for
//   every segment of the mixed batch -- decode rows, chunked-prefill rows and finetuning
//   forward-window rows [l_i, l_i+s) -- over keys [0, pos] held in KV
//   pages.  GQA is "packed": one CTA tile = 64 (query row, head-in-group) pairs that share a
//   KV head, so every K/V tile loaded from HBM serves the whole head group.  Keys may be
//   split across CTAs (flash-decoding); attn_combine_kernel merges the partials by LSE.
//   FT rows keep the natural-log LSE instead of the reference's per-row prob matrices
//   (tiny_model.hpp:102,149): that is the only softmax state that survives pruning.
// Backward (Alg. 2 lines 14-21): for the window's query
//   rows [a,b) at one layer, P is recomputed from Q, K and the saved LSE;
//   attn_bwd_dq_kernel produces dQ[a:b) (final), attn_bwd_dkdv_kernel adds this window's
//   dK/dV contributions over keys [0,b) into the fp32 ΔKVAccum (tiny_model.hpp:294-315).
// All matrix products use mma.sync m16n8k16 (bf16 in, fp32 accumulate); tiles are staged in
// XOR-swizzled shared memory with cp.async double buffering.
#include <cfloat>

#include <atomic>

#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"
#include "mma.cuh"

namespace cs {

namespace {
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

CS_DEV int page_row(const int* __restrict__ pt, int page_off, int j, int P) {
  return __ldg(pt + page_off + j / P) * P + (j % P);
}
}  // namespace

// ============================================================================ forward
template <int D>
__global__ void __launch_bounds__(128) attn_fwd_kernel(AttnFwdParams p) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  constexpr int BM = 64, BN = 64, CH = D / 8;
  constexpr int TILE = BN * D * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + BM * D * 2;
  uint8_t* sV = sK + 2 * TILE;

  const AttnWork w = p.work[blockIdx.x];
  const AttnSeg sg = p.segs[w.seg];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = p.grp;

  for (int idx = tid; idx < BM * CH; idx += 128) {
    const int r = idx / CH, c = idx % CH;
    const int qr = r / grp, g = r % grp;
    const __nv_bfloat16* src = p.q;
    int bytes = 0;
    if (qr < w.nq) {
      const long row = sg.q_start + w.q0 + qr;
      src = p.q + row * p.q_ld + (long)(w.kv_head * grp + g) * D + c * 8;
      bytes = 16;
    }
    cp_async16(smem_u32(sQ) + swz<D>(r, c), src, bytes);
  }
  cp_async_commit();

  const int kt0 = w.k_begin / BN;
  const int kt1 = (w.k_end + BN - 1) / BN;
  auto load_kv = [&](int kt, int stage) {
    for (int idx = tid; idx < BN * CH; idx += 128) {
      const int r = idx / CH, c = idx % CH;
      const int j = kt * BN + r;
      const __nv_bfloat16* ks = p.k_pool;
      const __nv_bfloat16* vs = p.v_pool;
      int bytes = 0;
      if (j < w.k_end) {
        const long off = (long)page_row(p.page_table, sg.page_off, j, p.page_size) * p.kv_dim +
                         w.kv_head * D + c * 8;
        ks += off;
        vs += off;
        bytes = 16;
      }
      cp_async16(smem_u32(sK + stage * TILE) + swz<D>(r, c), ks, bytes);
      cp_async16(smem_u32(sV + stage * TILE) + swz<D>(r, c), vs, bytes);
    }
  };
  if (kt0 < kt1) load_kv(kt0, 0);
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();

  uint32_t qf[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk)
    ldsm_x4(smem_u32(sQ) + swz<D>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)), qf[kk][0],
            qf[kk][1], qf[kk][2], qf[kk][3]);

  const int r_lo = warp * 16 + (lane >> 2), r_hi = r_lo + 8;
  const int qr_lo = r_lo / grp, qr_hi = r_hi / grp;
  const int pos_lo = qr_lo < w.nq ? sg.ctx_start + w.q0 + qr_lo : -1;
  const int pos_hi = qr_hi < w.nq ? sg.ctx_start + w.q0 + qr_hi : -1;

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

  for (int kt = kt0; kt < kt1; ++kt) {
    const int st = (kt - kt0) & 1;
    if (kt + 1 < kt1) load_kv(kt + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t kbase = smem_u32(sK + st * TILE), vbase = smem_u32(sV + st * TILE);

    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int nbp = 0; nbp < 4; ++nbp) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kbase + swz<D>(nbp * 16 + (lane & 7) + ((lane >> 4) << 3), kk * 2 + ((lane >> 3) & 1)),
                b0, b1, b2, b3);
        mma16816(s[2 * nbp], qf[kk], b0, b1);
        mma16816(s[2 * nbp + 1], qf[kk], b2, b3);
      }
    }
    // scale + causal/range mask
    float mx_lo = -INFINITY, mx_hi = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = kt * BN + nb * 8 + 2 * (lane & 3) + (e & 1);
        const int pos = e < 2 ? pos_lo : pos_hi;
        float v = s[nb][e] * p.scale_log2;
        if (j > pos || j >= w.k_end) v = -INFINITY;
        s[nb][e] = v;
      }
      mx_lo = fmaxf(mx_lo, fmaxf(s[nb][0], s[nb][1]));
      mx_hi = fmaxf(mx_hi, fmaxf(s[nb][2], s[nb][3]));
    }
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
    const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
    const float mu_lo = mn_lo == -INFINITY ? 0.f : mn_lo;
    const float mu_hi = mn_hi == -INFINITY ? 0.f : mn_hi;
    const float c_lo = exp2f(m_lo - mu_lo), c_hi = exp2f(m_hi - mu_hi);
    m_lo = mn_lo;
    m_hi = mn_hi;
    float rs_lo = 0.f, rs_hi = 0.f;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      s[nb][0] = exp2f(s[nb][0] - mu_lo);
      s[nb][1] = exp2f(s[nb][1] - mu_lo);
      s[nb][2] = exp2f(s[nb][2] - mu_hi);
      s[nb][3] = exp2f(s[nb][3] - mu_hi);
      rs_lo += s[nb][0] + s[nb][1];
      rs_hi += s[nb][2] + s[nb][3];
    }
    l_lo = l_lo * c_lo + rs_lo;
    l_hi = l_hi * c_hi + rs_hi;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= c_lo;
      o[i][1] *= c_lo;
      o[i][2] *= c_hi;
      o[i][3] *= c_hi;
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4];
      a[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      a[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      a[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      a[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vbase + swz<D>(kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), dp * 2 + (lane >> 4)),
                  b0, b1, b2, b3);
        mma16816(o[2 * dp], a, b0, b1);
        mma16816(o[2 * dp + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
  const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f;
  const float inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
  const float lse_lo = l_lo > 0.f ? (m_lo + __log2f(l_lo)) * kLn2 : -INFINITY;
  const float lse_hi = l_hi > 0.f ? (m_hi + __log2f(l_hi)) * kLn2 : -INFINITY;

#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = half ? r_hi : r_lo;
    const int qr = r / grp, g = r % grp;
    if (qr >= w.nq) continue;
    const float inv = half ? inv_hi : inv_lo;
    const float lse = half ? lse_hi : lse_lo;
    if (w.part < 0) {
      const long row = sg.q_start + w.q0 + qr;
      const int qh = w.kv_head * grp + g;
      __nv_bfloat16* dst = p.out + row * p.out_ld + (long)qh * D;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        const int d = i * 8 + 2 * (lane & 3);
        *reinterpret_cast<uint32_t*>(dst + d) =
            pack_bf16(o[i][2 * half] * inv, o[i][2 * half + 1] * inv);
      }
      if (p.lse && (lane & 3) == 0) p.lse[row * p.lse_ld + qh] = lse;
    } else {
      float* dst = p.part_o + ((long)w.part * BM + r) * D;
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        const int d = i * 8 + 2 * (lane & 3);
        *reinterpret_cast<float2*>(dst + d) =
            make_float2(o[i][2 * half] * inv, o[i][2 * half + 1] * inv);
      }
      if ((lane & 3) == 0) p.part_lse[(long)w.part * BM + r] = lse;
    }
  }
}

// Merge split-KV partials: o = sum_s o_s * exp(lse_s - lse), lse = log sum_s exp(lse_s).
// One warp per packed row (lanes over d, 4 columns each), one pass with a running max: the
// part loads are independent of the merge arithmetic, so a row costs one memory round trip
// (the two-pass max-then-sum form was two dependent round trips per row).
template <int D>
__global__ void __launch_bounds__(128) attn_combine_kernel(AttnFwdParams p) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  // launched with PDL: the CTAs are resident while the producing attention kernel drains;
  // its partials are visible after the wait
  griddep_wait();
  const AttnCombine c = p.combine[blockIdx.x];
  const AttnSeg sg = p.segs[c.seg];
  const int grp = p.grp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = lane * 4;
  // blockIdx.y: 16-row slice of the item (a 256-row tcgen05 part needs 16 CTAs: one CTA per
  // item left the merge latency-bound)
  const int r_end = min(c.nq * grp, (int)(blockIdx.y + 1) * 16);
  for (int r = blockIdx.y * 16 + warp; r < r_end; r += 4) {
    float mx = -INFINITY, den = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < c.n_parts; s0 += 4) {
      float l[4];
      float4 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // issue the group's loads before any arithmetic
        const long pr = (long)(c.part0 + min(s0 + i, c.n_parts - 1)) * p.part_rows + r;
        l[i] = s0 + i < c.n_parts ? __ldg(p.part_lse + pr) : -INFINITY;
        v[i] = __ldg(reinterpret_cast<const float4*>(p.part_o + pr * D + (d & (D - 1))));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (l[i] > -INFINITY) {  // an empty part (no unmasked key) contributes nothing
          const float nm = fmaxf(mx, l[i]);
          const float a = __expf(mx - nm), b = __expf(l[i] - nm);
          den = den * a + b;
          acc.x = acc.x * a + b * v[i].x;
          acc.y = acc.y * a + b * v[i].y;
          acc.z = acc.z * a + b * v[i].z;
          acc.w = acc.w * a + b * v[i].w;
          mx = nm;
        }
      }
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    const int qr = r / grp, g = r - qr * grp;
    const long row = sg.q_start + c.q0 + qr;
    const int qh = c.kv_head * grp + g;
    if (d < D) {
      bf16* dst = p.out + row * p.out_ld + (long)qh * D + d;
      *reinterpret_cast<uint32_t*>(dst) = pack_bf16(acc.x * inv, acc.y * inv);
      *reinterpret_cast<uint32_t*>(dst + 2) = pack_bf16(acc.z * inv, acc.w * inv);
    }
    if (lane == 0 && p.lse) p.lse[row * p.lse_ld + qh] = den > 0.f ? mx + __logf(den) : -INFINITY;
  }
}

// delta[r, h] = sum_d dO[r, h, d] * O[r, h, d]: an 8-lane group per (row, head) pair, 16-byte
// loads (8 bf16) per lane, 3-shuffle group reduction
__global__ void attn_bwd_delta_kernel(const __nv_bfloat16* __restrict__ dO, long do_ld,
                                      const __nv_bfloat16* __restrict__ O, long o_ld, int rows,
                                      int heads, int D, float* __restrict__ delta) {
  const long pair = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;
  const bool ok = pair < (long)rows * heads;  // (no early exit: the group shuffles use all lanes)
  const int r = ok ? (int)(pair / heads) : 0, h = ok ? (int)(pair % heads) : 0;
  const __nv_bfloat16* a = dO + (long)r * do_ld + (long)h * D;
  const __nv_bfloat16* b = O + (long)r * o_ld + (long)h * D;
  float acc = 0.f;
  for (int d = sub * 8; ok && d < D; d += 64) {
    const uint4 x = *reinterpret_cast<const uint4*>(a + d);
    const uint4 y = *reinterpret_cast<const uint4*>(b + d);
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 u = __bfloat1622float2(x2[q]), v = __bfloat1622float2(y2[q]);
      acc += u.x * v.x + u.y * v.y;
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  if (ok && sub == 0) delta[(long)r * heads + h] = acc;
}

// dQ for query tiles of the window: CTA = (64 packed rows, kv head); loop over key tiles [0, b)
template <int D>
__global__ void __launch_bounds__(128) attn_bwd_dq_kernel(AttnBwdParams p) {
  constexpr int BM = 64, BN = 64, CH = D / 8, TILE = BN * D * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sO = sQ + BM * D * 2;  // dO
  uint8_t* sK = sO + BM * D * 2;
  uint8_t* sV = sK + 2 * TILE;
  const int grp = p.grp;
  const int rows_per_tile = BM / grp;
  const int q0 = blockIdx.x * rows_per_tile;  // window-local first row
  const int kvh = blockIdx.y;
  const int nq = min(rows_per_tile, p.b - p.a - q0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int idx = tid; idx < BM * CH; idx += 128) {
    const int r = idx / CH, c = idx % CH;
    const int qr = r / grp, g = r % grp;
    const __nv_bfloat16* sq = p.q_cache;
    const __nv_bfloat16* so = p.dO;
    int bytes = 0;
    if (qr < nq) {
      const int qh = kvh * grp + g;
      sq = p.q_cache + (long)(p.a + q0 + qr) * p.q_ld + (long)qh * D + c * 8;
      so = p.dO + (long)(q0 + qr) * p.do_ld + (long)qh * D + c * 8;
      bytes = 16;
    }
    cp_async16(smem_u32(sQ) + swz<D>(r, c), sq, bytes);
    cp_async16(smem_u32(sO) + swz<D>(r, c), so, bytes);
  }
  cp_async_commit();
  const int kt1 = (p.a + q0 + nq + BN - 1) / BN;  // keys [0, last position]
  auto load_kv = [&](int kt, int stage) {
    for (int idx = tid; idx < BN * CH; idx += 128) {
      const int r = idx / CH, c = idx % CH;
      const int j = kt * BN + r;
      const __nv_bfloat16* ks = p.k_pool;
      const __nv_bfloat16* vs = p.v_pool;
      int bytes = 0;
      if (j < p.b) {
        const long off =
            (long)page_row(p.page_table, p.page_off, j, p.page_size) * p.kv_dim + kvh * D + c * 8;
        ks += off;
        vs += off;
        bytes = 16;
      }
      cp_async16(smem_u32(sK + stage * TILE) + swz<D>(r, c), ks, bytes);
      cp_async16(smem_u32(sV + stage * TILE) + swz<D>(r, c), vs, bytes);
    }
  };
  load_kv(0, 0);
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();

  uint32_t qf[D / 16][4], of[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const uint32_t off = swz<D>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4));
    ldsm_x4(smem_u32(sQ) + off, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
    ldsm_x4(smem_u32(sO) + off, of[kk][0], of[kk][1], of[kk][2], of[kk][3]);
  }
  const int r_lo = warp * 16 + (lane >> 2), r_hi = r_lo + 8;
  float lse2[2], dlt[2];
  int pos[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = h ? r_hi : r_lo;
    const int qr = r / grp, g = r % grp;
    if (qr < nq) {
      const int qh = kvh * grp + g;
      pos[h] = p.a + q0 + qr;
      lse2[h] = p.lse[(long)pos[h] * p.lse_ld + qh] * kLog2e;
      dlt[h] = p.delta[(long)(q0 + qr) * p.delta_ld + qh];
    } else {
      pos[h] = -1;
      lse2[h] = 0.f;
      dlt[h] = 0.f;
    }
  }
  float dq[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int kt = 0; kt < kt1; ++kt) {
    const int st = kt & 1;
    if (kt + 1 < kt1) load_kv(kt + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t kbase = smem_u32(sK + st * TILE), vbase = smem_u32(sV + st * TILE);
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      s[i][0] = s[i][1] = s[i][2] = s[i][3] = dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int nbp = 0; nbp < 4; ++nbp) {
        const uint32_t off =
            swz<D>(nbp * 16 + (lane & 7) + ((lane >> 4) << 3), kk * 2 + ((lane >> 3) & 1));
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kbase + off, b0, b1, b2, b3);
        mma16816(s[2 * nbp], qf[kk], b0, b1);
        mma16816(s[2 * nbp + 1], qf[kk], b2, b3);
        ldsm_x4(vbase + off, b0, b1, b2, b3);
        mma16816(dp[2 * nbp], of[kk], b0, b1);
        mma16816(dp[2 * nbp + 1], of[kk], b2, b3);
      }
    }
    // P = exp2(s*scale_log2 - lse2) ; dS = P * (dP - Delta)
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = e >> 1;
        const int j = kt * BN + nb * 8 + 2 * (lane & 3) + (e & 1);
        float pv = (j <= pos[h] && j < p.b) ? exp2f(s[nb][e] * p.scale_log2 - lse2[h]) : 0.f;
        s[nb][e] = pv * (dp[nb][e] - dlt[h]);
      }
    }
    // dQ += dS . K   (K as B operand with k = key, n = d -> transposed ldmatrix)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4];
      a[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      a[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      a[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      a[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dpi = 0; dpi < D / 16; ++dpi) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(kbase + swz<D>(kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), dpi * 2 + (lane >> 4)),
                  b0, b1, b2, b3);
        mma16816(dq[2 * dpi], a, b0, b1);
        mma16816(dq[2 * dpi + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = h ? r_hi : r_lo;
    const int qr = r / grp, g = r % grp;
    if (qr >= nq) continue;
    float* dst = p.dq + (long)(q0 + qr) * p.dq_ld + (long)(kvh * grp + g) * D;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int d = i * 8 + 2 * (lane & 3);
      *reinterpret_cast<float2*>(dst + d) =
          make_float2(dq[i][2 * h] * p.scale, dq[i][2 * h + 1] * p.scale);
    }
  }
}

// dK/dV for one key tile (64 keys, 16 per warp) and one kv head; loop over the window's
// query tiles; result added into ΔKVAccum rows of the tile.
template <int D>
__global__ void __launch_bounds__(128, 1) attn_bwd_dkdv_kernel(AttnBwdParams p) {
  constexpr int BM = 64, BN = 64, CH = D / 8, TILE = BM * D * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sK = smem;
  uint8_t* sV = sK + BN * D * 2;
  uint8_t* sQ = sV + BN * D * 2;  // 2 stages
  uint8_t* sO = sQ + 2 * TILE;    // 2 stages (dO)
  float* sL = reinterpret_cast<float*>(sO + 2 * TILE);  // [2][BM] lse2
  float* sD = sL + 2 * BM;                               // [2][BM] delta
  int* sP = reinterpret_cast<int*>(sD + 2 * BM);        // [2][BM] position (-1 invalid)

  const int grp = p.grp;
  const int rows_per_tile = BM / grp;
  const int k0 = blockIdx.x * BN;
  const int kvh = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int idx = tid; idx < BN * CH; idx += 128) {
    const int r = idx / CH, c = idx % CH;
    const int j = k0 + r;
    const __nv_bfloat16* ks = p.k_pool;
    const __nv_bfloat16* vs = p.v_pool;
    int bytes = 0;
    if (j < p.b) {
      const long off =
          (long)page_row(p.page_table, p.page_off, j, p.page_size) * p.kv_dim + kvh * D + c * 8;
      ks += off;
      vs += off;
      bytes = 16;
    }
    cp_async16(smem_u32(sK) + swz<D>(r, c), ks, bytes);
    cp_async16(smem_u32(sV) + swz<D>(r, c), vs, bytes);
  }
  cp_async_commit();

  // query tiles whose last position >= k0
  const int nrows = p.b - p.a;
  const int n_qt = (nrows + rows_per_tile - 1) / rows_per_tile;
  int qt_begin = 0;
  if (k0 > p.a) qt_begin = (k0 - p.a) / rows_per_tile;
  auto load_q = [&](int qt, int stage) {
    const int q0 = qt * rows_per_tile;
    const int nq = min(rows_per_tile, nrows - q0);
    for (int idx = tid; idx < BM * CH; idx += 128) {
      const int r = idx / CH, c = idx % CH;
      const int qr = r / grp, g = r % grp;
      const __nv_bfloat16* sq = p.q_cache;
      const __nv_bfloat16* so = p.dO;
      int bytes = 0;
      if (qr < nq) {
        const int qh = kvh * grp + g;
        sq = p.q_cache + (long)(p.a + q0 + qr) * p.q_ld + (long)qh * D + c * 8;
        so = p.dO + (long)(q0 + qr) * p.do_ld + (long)qh * D + c * 8;
        bytes = 16;
      }
      cp_async16(smem_u32(sQ + stage * TILE) + swz<D>(r, c), sq, bytes);
      cp_async16(smem_u32(sO + stage * TILE) + swz<D>(r, c), so, bytes);
    }
    for (int r = tid; r < BM; r += 128) {
      const int qr = r / grp, g = r % grp;
      if (qr < nq) {
        const int qh = kvh * grp + g;
        const int pos = p.a + q0 + qr;
        sL[stage * BM + r] = p.lse[(long)pos * p.lse_ld + qh] * kLog2e;
        sD[stage * BM + r] = p.delta[(long)(q0 + qr) * p.delta_ld + qh];
        sP[stage * BM + r] = pos;
      } else {
        sL[stage * BM + r] = 0.f;
        sD[stage * BM + r] = 0.f;
        sP[stage * BM + r] = -1;
      }
    }
  };

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
    dk[i][0] = dk[i][1] = dk[i][2] = dk[i][3] = dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;

  const int key_lo = k0 + warp * 16 + (lane >> 2), key_hi = key_lo + 8;
  if (qt_begin < n_qt) load_q(qt_begin, 0);
  cp_async_commit();

  for (int qt = qt_begin; qt < n_qt; ++qt) {
    const int st = (qt - qt_begin) & 1;
    if (qt + 1 < n_qt) load_q(qt + 1, st ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t qbase = smem_u32(sQ + st * TILE), obase = smem_u32(sO + st * TILE);
    const float* L2 = sL + st * BM;
    const float* DL = sD + st * BM;
    const int* PS = sP + st * BM;
    // S^T = K_w Q^T and dP^T = V_w dO^T : [16 keys x 64 packed rows]
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      s[i][0] = s[i][1] = s[i][2] = s[i][3] = dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ka[4], va[4];
      const uint32_t aoff = swz<D>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4));
      ldsm_x4(smem_u32(sK) + aoff, ka[0], ka[1], ka[2], ka[3]);
      ldsm_x4(smem_u32(sV) + aoff, va[0], va[1], va[2], va[3]);
#pragma unroll
      for (int nbp = 0; nbp < 4; ++nbp) {
        const uint32_t off =
            swz<D>(nbp * 16 + (lane & 7) + ((lane >> 4) << 3), kk * 2 + ((lane >> 3) & 1));
        uint32_t b0, b1, b2, b3;
        ldsm_x4(qbase + off, b0, b1, b2, b3);
        mma16816(s[2 * nbp], ka, b0, b1);
        mma16816(s[2 * nbp + 1], ka, b2, b3);
        ldsm_x4(obase + off, b0, b1, b2, b3);
        mma16816(dp[2 * nbp], va, b0, b1);
        mma16816(dp[2 * nbp + 1], va, b2, b3);
      }
    }
    // P^T, dS^T (element (key, packed row)); rows index columns here
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = (e < 2) ? key_lo : key_hi;
        const int r = nb * 8 + 2 * (lane & 3) + (e & 1);
        const int pos = PS[r];
        const float pv =
            (pos >= 0 && key <= pos && key < p.b) ? exp2f(s[nb][e] * p.scale_log2 - L2[r]) : 0.f;
        s[nb][e] = pv;
        dp[nb][e] = pv * (dp[nb][e] - DL[r]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q   (B operands: k = packed row, n = d -> transposed ldmatrix)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4], da[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
      da[0] = pack_bf16(dp[2 * kk][0], dp[2 * kk][1]);
      da[1] = pack_bf16(dp[2 * kk][2], dp[2 * kk][3]);
      da[2] = pack_bf16(dp[2 * kk + 1][0], dp[2 * kk + 1][1]);
      da[3] = pack_bf16(dp[2 * kk + 1][2], dp[2 * kk + 1][3]);
#pragma unroll
      for (int dpi = 0; dpi < D / 16; ++dpi) {
        const uint32_t off =
            swz<D>(kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), dpi * 2 + (lane >> 4));
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(obase + off, b0, b1, b2, b3);
        mma16816(dv[2 * dpi], pa, b0, b1);
        mma16816(dv[2 * dpi + 1], pa, b2, b3);
        ldsm_x4_t(qbase + off, b0, b1, b2, b3);
        mma16816(dk[2 * dpi], da, b0, b1);
        mma16816(dk[2 * dpi + 1], da, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  // ΔKVAccum rows [k0 + warp*16 ..] += contributions (this CTA owns them: no atomics)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int key = h ? key_hi : key_lo;
    if (key >= p.b) continue;
    float* ak = p.dk_acc + (long)key * p.acc_ld + kvh * D;
    float* av = p.dv_acc + (long)key * p.acc_ld + kvh * D;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int d = i * 8 + 2 * (lane & 3);
      float2 x = *reinterpret_cast<float2*>(ak + d);
      x.x += dk[i][2 * h] * p.scale;
      x.y += dk[i][2 * h + 1] * p.scale;
      *reinterpret_cast<float2*>(ak + d) = x;
      float2 y = *reinterpret_cast<float2*>(av + d);
      y.x += dv[i][2 * h];
      y.y += dv[i][2 * h + 1];
      *reinterpret_cast<float2*>(av + d) = y;
    }
  }
}

// ============================================================================ launchers
namespace {
template <typename K>
cudaError_t set_smem(K kern, int bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
}  // namespace

cudaError_t attn_fwd(const AttnFwdParams& p, int head_dim, int n_work, int n_combine,
                     cudaStream_t st) {
  // the combine also merges the decode kernel's partials (attn_decode runs first)
  if (n_work <= 0 && n_combine <= 0) return cudaSuccess;
  if (head_dim == 128) {
    constexpr int smem = 64 * 128 * 2 * 5;
    static bool once = (set_smem(attn_fwd_kernel<128>, smem), true);
    (void)once;
    if (n_work > 0) {
      cs::g_launches.fetch_add(1, std::memory_order_relaxed);
      attn_fwd_kernel<128><<<n_work, 128, smem, st>>>(p);
    }
    if (n_combine > 0) {
      cs::g_launches.fetch_add(1, std::memory_order_relaxed);
      const cudaError_t e = launch_pdl(attn_combine_kernel<128>, dim3(n_combine, p.comb_slices), dim3(128), 0, st, p);
      if (e != cudaSuccess) return e;
    }
  } else if (head_dim == 64) {
    constexpr int smem = 64 * 64 * 2 * 5;
    static bool once = (set_smem(attn_fwd_kernel<64>, smem), true);
    (void)once;
    if (n_work > 0) {
      cs::g_launches.fetch_add(1, std::memory_order_relaxed);
      attn_fwd_kernel<64><<<n_work, 128, smem, st>>>(p);
    }
    if (n_combine > 0) {
      cs::g_launches.fetch_add(1, std::memory_order_relaxed);
      const cudaError_t e = launch_pdl(attn_combine_kernel<64>, dim3(n_combine, p.comb_slices), dim3(128), 0, st, p);
      if (e != cudaSuccess) return e;
    }
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t attn_combine(const AttnFwdParams& p, int head_dim, int n_combine, cudaStream_t st) {
  if (n_combine <= 0) return cudaSuccess;
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  const dim3 grid(n_combine, (p.part_rows + 15) / 16);
  if (head_dim == 128) return launch_pdl(attn_combine_kernel<128>, grid, dim3(128), 0, st, p);
  if (head_dim == 64) return launch_pdl(attn_combine_kernel<64>, grid, dim3(128), 0, st, p);
  return cudaErrorInvalidValue;
  return cudaGetLastError();
}

void attn_bwd_delta_kernel_launch(const AttnBwdParams& p, int rows, int n_heads, cudaStream_t st) {
  const long threads = (long)rows * n_heads * 8;  // 8 lanes per (row, head)
  attn_bwd_delta_kernel<<<(int)((threads + 255) / 256), 256, 0, st>>>(p.dO, p.do_ld, p.O, p.o_ld, rows,
                                                                     n_heads, p.q_ld / n_heads, p.delta);
}

cudaError_t attn_bwd(const AttnBwdParams& p, int head_dim, int n_heads, cudaStream_t st) {
  const int rows = p.b - p.a;
  if (rows <= 0) return cudaSuccess;
  {
    const long threads = (long)rows * n_heads * 8;  // 8 lanes per (row, head)
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    attn_bwd_delta_kernel<<<(int)((threads + 255) / 256), 256, 0, st>>>(
        p.dO, p.do_ld, p.O, p.o_ld, rows, n_heads, head_dim, p.delta);
  }
  const int rows_per_tile = 64 / p.grp;
  dim3 gq((rows + rows_per_tile - 1) / rows_per_tile, n_heads / p.grp);
  dim3 gk((p.b + 63) / 64, n_heads / p.grp);
  if (head_dim == 128) {
    constexpr int sq = 64 * 128 * 2 * 6;
    constexpr int sk = 64 * 128 * 2 * 6 + 64 * 4 * 6;
    static bool once = (set_smem(attn_bwd_dq_kernel<128>, sq),
                        set_smem(attn_bwd_dkdv_kernel<128>, sk), true);
    (void)once;
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    attn_bwd_dq_kernel<128><<<gq, 128, sq, st>>>(p);
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    attn_bwd_dkdv_kernel<128><<<gk, 128, sk, st>>>(p);
  } else if (head_dim == 64) {
    constexpr int sq = 64 * 64 * 2 * 6;
    constexpr int sk = 64 * 64 * 2 * 6 + 64 * 4 * 6;
    static bool once = (set_smem(attn_bwd_dq_kernel<64>, sq),
                        set_smem(attn_bwd_dkdv_kernel<64>, sk), true);
    (void)once;
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    attn_bwd_dq_kernel<64><<<gq, 128, sq, st>>>(p);
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    attn_bwd_dkdv_kernel<64><<<gk, 128, sk, st>>>(p);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cs
