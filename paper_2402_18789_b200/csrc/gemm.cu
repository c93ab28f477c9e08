// gemm.cu -- K1/K3/K10: the base-model GEMMs of the co-serving step on sm_100a.
//
//   C[M,N] (op)= A[M,K] . B[N,K]^T      A, B bf16 K-major (row-major with K contiguous),
//                                        fp32 accumulation in TMEM.
// Replaces the reference's naive f64 `matmul` / `matmul_nt` (matrix.hpp:69-105) on every
// projection of tiny_model.hpp:196-211 (forward, B = W^T stored [out,in]) and :283-319
// (token-level backward dX = dY.W^T, B = W in the reference's own [in,out] layout).
//
// Design (one CTA per SM, persistent over a static tile list):
//   warp 0      : TMA producer  (cp.async.bulk.tensor 2D, SWIZZLE_128B, mbarrier complete_tx)
//   warp 1      : MMA issuer    (one thread issues tcgen05.mma.cta_group::1.kind::f16,
//                                M=128, N=BN, K=16 per instruction; commits to mbarriers)
//   warp 2      : TMEM allocator (2*BN columns: double-buffered accumulator)
//   warps 4..7  : epilogue      (tcgen05.ld 32x32b -> registers -> bias/residual -> global)
// Work unit = (m block, n block, k split).  Split-K partial sums are combined with fp32
// vector atomics (only for fp32 outputs).  Rows >= M / cols >= N are masked in the
// epilogue, so A/B tensor maps can describe whole (capacity-sized) buffers.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include <atomic>

#include "common.cuh"
#include "kernels.h"

namespace cs {

struct GemmArgs {
  int M, N, K;
  int kb_total;  // ceil(K / 64)
  int splits;
  int num_m, num_n;
  int epi;
  void* C;
  long ldc;
  const float* bias;
  int b_const;  // B is not written by the previous kernel on the stream (weights): its first
                // stages may be fetched before griddepcontrol.wait
  GemmScatter sc;  // EPI_F32_SCATTER destination (peer staging slots)
  int b_mn;        // 1: B stored [K rows][N cols] (N contiguous): MN-major B operand
  // tail split (CTA-pair kernel, accumulating epilogues): work units [0, full_units) are whole
  // tiles, the tiles after them are split `splits` ways along K -- only the last, partial wave
  // is split, so it is spread over all pairs instead of idling most of them.  0: uniform splits
  int full_units = 0;
  int units = 0;  // total work units
  void* C2 = nullptr;  // EPI_SWIGLU (kernels.h)
  long ldc2 = 0;
  int c2_row0 = 0;
  int m_cols = 0;
  QkvEpi qkv;          // EPI_QKV_ROPE
  int group_m = 1;     // m-blocks per raster run (tile_mn)
};

// SM (small M <= 64): only 64 rows of A are loaded per stage; the M=128 MMA reads the other 64
// rows from whatever follows in shared memory and those accumulator rows are never stored.  The
// freed 8 KB per stage go to more weight (B) stages in flight -- small-M GEMMs are weight
// streams, bounded by the bytes each SM keeps in flight.
template <int BN, bool SM = false>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;
  static constexpr int A_ROWS = SM ? 64 : 128;
  static constexpr int A_BYTES = A_ROWS * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (196 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = (2 * BN) < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int CHUNK = BN >= 32 ? 32 : 16;
};

// tile index -> (m, n) block, grouped raster: runs of group_m m-blocks sweep all n-blocks, so
// the tiles in flight at once (a wave of 74 pairs / 148 CTAs) share A rows and B columns in L2
// (M = 8192 backward dX GEMMs: a plain m-fastest order kept all 32 m-blocks' A rows in flight,
// 1394 vs cuBLAS 1612 TF/s at K = 28672), and every run streams B (the weights) once: the host
// sizes the runs evenly (<= 12 m-blocks) -- a ragged last run of one m-block re-read all of B
// (gate||up M = 1088 on 128-row tiles: 217 us vs 191 us)
__device__ __forceinline__ void tile_mn(int t, const GemmArgs& a, int& m, int& n) {
  const int G = a.group_m;
  const int per = G * a.num_n;
  const int g = t / per, r = t - g * per;
  const int gm = min(G, a.num_m - g * G);
  m = g * G + r % gm;
  n = r / gm;
}
inline int group_m_for(int num_m) {
  const int ng = (num_m + 11) / 12;
  return (num_m + ng - 1) / ng;
}

__device__ __forceinline__ void decode_work(int w, const GemmArgs& a, int& m_blk, int& n_blk,
                                            int& kb0, int& kb1) {
  if (a.full_units > 0) {
    int t = w, ks = 0, sp = 1;
    if (w >= a.full_units) {
      const int u = w - a.full_units;
      t = a.full_units + u / a.splits;
      ks = u % a.splits;
      sp = a.splits;
    }
    tile_mn(t, a, m_blk, n_blk);
    kb0 = (int)(((long)ks * a.kb_total) / sp);
    kb1 = (int)(((long)(ks + 1) * a.kb_total) / sp);
    return;
  }
  // uniform K split: every tile's split ks, then split ks + 1 -- the units of one split run
  // together, so a wave shares each A slice across the n-blocks and each B slice across the
  // m-blocks in L2 (the LM head's dH = dlogits U, K = V: with the splits of a tile adjacent a
  // wave needed all of A's slices and re-read A once per ~2 n-blocks)
  const long tiles = (long)a.num_m * a.num_n;
  const int ks = (int)(w / tiles);
  tile_mn((int)(w % tiles), a, m_blk, n_blk);
  kb0 = (int)(((long)ks * a.kb_total) / a.splits);
  kb1 = (int)(((long)(ks + 1) * a.kb_total) / a.splits);
}

template <int BN>
__device__ __forceinline__ void epilogue_store(const GemmArgs& a, int row, int col0,
                                               const uint32_t* r, int cnt) {
  // r: cnt fp32 values (as bits) for columns col0 .. col0+cnt-1 of `row`
  if (row >= a.M) return;
  const bool full = (col0 + cnt) <= a.N;
  if (a.epi == EPI_BF16) {
    __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(a.C) + (long)row * a.ldc + col0;
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < cnt) v[i] = __uint_as_float(r[i]) + (a.bias ? a.bias[min(col0 + i, a.N - 1)] : 0.f);
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        if (i < cnt) {
          uint4 p;
          p.x = pack_bf16(v[i], v[i + 1]);
          p.y = pack_bf16(v[i + 2], v[i + 3]);
          p.z = pack_bf16(v[i + 4], v[i + 5]);
          p.w = pack_bf16(v[i + 6], v[i + 7]);
          *reinterpret_cast<uint4*>(C + i) = p;
        }
      }
    } else {
      for (int i = 0; i < cnt; ++i)
        if (col0 + i < a.N) C[i] = __float2bfloat16(v[i]);
    }
  } else {
    float* C;
    if (a.epi == EPI_F32_SCATTER) {  // fused TP all-reduce: partial -> owner's staging slot
      const int rpo = a.sc.rows_per_owner, owner = row / rpo;
      C = a.sc.peer[owner] + ((long)a.sc.rank * rpo + (row - owner * rpo)) * a.ldc + col0;
    } else {
      C = reinterpret_cast<float*>(a.C) + (long)row * a.ldc + col0;
    }
    const bool atomic = a.splits > 1 || a.epi == EPI_F32_ATOMIC;
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        if (i < cnt) {
          float4 v = make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                 __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
          float4* p = reinterpret_cast<float4*>(C + i);
          if (atomic) {
            atomicAdd(p, v);
          } else if (a.epi == EPI_F32_ADD) {
            float4 o = *p;
            o.x += v.x; o.y += v.y; o.z += v.z; o.w += v.w;
            *p = o;
          } else {
            *p = v;
          }
        }
      }
    } else {
      for (int i = 0; i < cnt; ++i) {
        if (col0 + i >= a.N) break;
        float v = __uint_as_float(r[i]);
        if (atomic) atomicAdd(C + i, v);
        else if (a.epi == EPI_F32_ADD) C[i] += v;
        else C[i] = v;
      }
    }
  }
}

// EPI_SWIGLU: 32 gate columns (g, output columns col_g .. col_g+31, inside the gate half of a
// 128-column group) and the matching 32 up columns (64 further).  Rounding points as the
// unfused path (tiny_model.hpp:205 in the LLaMA generalisation): g and u rounded to bf16, then
// m = bf16(silu(g) * u) in fp32.
__device__ __forceinline__ void epilogue_swiglu(const GemmArgs& a, int row, int col_g, const uint32_t* g,
                                                const uint32_t* u) {
  if (row >= a.M || col_g >= a.N) return;
  uint32_t gp[16], up[16], mp[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    gp[i] = pack_bf16(__uint_as_float(g[2 * i]), __uint_as_float(g[2 * i + 1]));
    up[i] = pack_bf16(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]));
    const __nv_bfloat162 gb = *reinterpret_cast<const __nv_bfloat162*>(&gp[i]);
    const __nv_bfloat162 ub = *reinterpret_cast<const __nv_bfloat162*>(&up[i]);
    const float g0 = __low2float(gb), g1 = __high2float(gb);
    const float s0 = g0 * __fdividef(1.f, 1.f + __expf(-g0)), s1 = g1 * __fdividef(1.f, 1.f + __expf(-g1));
    mp[i] = pack_bf16(s0 * __low2float(ub), s1 * __high2float(ub));
  }
  const int f0 = (col_g >> 7) * 64 + (col_g & 127);
  __nv_bfloat16* m = reinterpret_cast<__nv_bfloat16*>(a.C) + (long)row * a.ldc;
#pragma unroll
  for (int i = 0; i < 16; i += 4)
    *reinterpret_cast<uint4*>(m + f0 + 2 * i) = make_uint4(mp[i], mp[i + 1], mp[i + 2], mp[i + 3]);
  if (f0 + 32 == a.m_cols)  // the K-concatenation pad columns of m (LoRA-up inputs, lora_pack)
    for (int c = a.m_cols; c < a.ldc; c += 8)
      *reinterpret_cast<uint4*>(m + c) = make_uint4(0, 0, 0, 0);
  if (a.C2 && row >= a.c2_row0) {
    __nv_bfloat16* s = reinterpret_cast<__nv_bfloat16*>(a.C2) + (long)(row - a.c2_row0) * a.ldc2 + col_g;
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
      *reinterpret_cast<uint4*>(s + 2 * i) = make_uint4(gp[i], gp[i + 1], gp[i + 2], gp[i + 3]);
      *reinterpret_cast<uint4*>(s + 64 + 2 * i) = make_uint4(up[i], up[i + 1], up[i + 2], up[i + 3]);
    }
  }
}

// EPI_QKV_ROPE: one 128-column head group (head-aligned, output columns col .. col+127) of `row`,
// read from TMEM in 32-column chunks (tb = this row's lane, this group's first column).
// q / k heads: rotate-half pairs (i, i+64) of RoPE; q stays in C (and the FT rows' q_cache),
// k and v go to the row's page slot of the K / V pool (tiny_model.hpp:225-232 + paging).
__device__ __forceinline__ void epilogue_qkv_rope(const GemmArgs& a, int row, int col, uint32_t tb, long prow,
                                                  int pos) {
  const QkvEpi& e = a.qkv;
  const bool valid = row < a.M && col < a.N;
  const bool isq = col < e.q_dim, isk = !isq && col < e.q_dim + e.kv_dim;
  __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(a.C) + (long)row * a.ldc;
  if (isq || isk) {
#pragma unroll 1
    for (int h = 0; h < 64; h += 32) {
      uint32_t x1[32], x2[32];
      tmem_ld_32x32b_x32(tb + h, x1);
      tmem_ld_32x32b_x32(tb + 64 + h, x2);
      tmem_ld_wait();
      if (!valid) continue;
      uint32_t o1[16], o2[16];
      const float2* tab = e.rope_tab + (long)pos * 64 + h;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        float v1[2], v2[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int c = col + h + j + t;
          v1[t] = __bfloat162float(__float2bfloat16(__uint_as_float(x1[j + t]) + (a.bias ? a.bias[c] : 0.f)));
          v2[t] = __bfloat162float(__float2bfloat16(__uint_as_float(x2[j + t]) + (a.bias ? a.bias[c + 64] : 0.f)));
          if (e.use_rope) {
            const float2 cs = tab[j + t];
            const float r1 = v1[t] * cs.x - v2[t] * cs.y, r2 = v2[t] * cs.x + v1[t] * cs.y;
            v1[t] = r1;
            v2[t] = r2;
          }
        }
        o1[j >> 1] = pack_bf16(v1[0], v1[1]);
        o2[j >> 1] = pack_bf16(v2[0], v2[1]);
      }
      __nv_bfloat16* d1;
      if (isq) {
        d1 = C + col + h;
      } else {
        d1 = e.k_pool + prow * e.kv_dim + (col - e.q_dim) + h;
      }
#pragma unroll
      for (int i = 0; i < 16; i += 4) {
        *reinterpret_cast<uint4*>(d1 + 2 * i) = make_uint4(o1[i], o1[i + 1], o1[i + 2], o1[i + 3]);
        *reinterpret_cast<uint4*>(d1 + 64 + 2 * i) = make_uint4(o2[i], o2[i + 1], o2[i + 2], o2[i + 3]);
      }
      if (isq && e.q_cache && row >= e.ft_row0) {
        __nv_bfloat16* qc = e.q_cache + (long)pos * e.q_dim + col + h;
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          *reinterpret_cast<uint4*>(qc + 2 * i) = make_uint4(o1[i], o1[i + 1], o1[i + 2], o1[i + 3]);
          *reinterpret_cast<uint4*>(qc + 64 + 2 * i) = make_uint4(o2[i], o2[i + 1], o2[i + 2], o2[i + 3]);
        }
      }
    }
  } else {  // v head -> the V page slot
#pragma unroll 1
    for (int h = 0; h < 128; h += 32) {
      uint32_t x[32];
      tmem_ld_32x32b_x32(tb + h, x);
      tmem_ld_wait();
      if (!valid) continue;
      uint32_t o[16];
#pragma unroll
      for (int j = 0; j < 32; j += 2)
        o[j >> 1] = pack_bf16(__uint_as_float(x[j]) + (a.bias ? a.bias[col + h + j] : 0.f),
                              __uint_as_float(x[j + 1]) + (a.bias ? a.bias[col + h + j + 1] : 0.f));
      __nv_bfloat16* d = e.v_pool + prow * e.kv_dim + (col - e.q_dim - e.kv_dim) + h;
#pragma unroll
      for (int i = 0; i < 16; i += 4) *reinterpret_cast<uint4*>(d + 2 * i) = make_uint4(o[i], o[i + 1], o[i + 2], o[i + 3]);
    }
  }
}

// the row's page slot and position for EPI_QKV_ROPE (one lookup per row and tile)
__device__ __forceinline__ void qkv_row_slot(const GemmArgs& a, int row, long& prow, int& pos) {
  prow = 0;
  pos = 0;
  if (row >= a.M) return;
  pos = __ldg(a.qkv.row_pos + row);
  prow = __ldg(a.qkv.row_slot + row);
}

// B stage of BN columns x 64 K: K-major = one box {64 K, BN rows}; MN-major (B stored
// [K][N]) = BN/64 boxes {64 N, 64 K rows}, 8 KB apart
template <int BN>
__device__ __forceinline__ void load_b(const CUtensorMap* tmB, uint64_t* bar, uint8_t* sb, int kb, int n0,
                                       int b_mn) {
  if (!b_mn) {
    tma_load_2d(tmB, bar, sb, kb * 64, n0);
  } else {
#pragma unroll
    for (int c = 0; c < BN / 64; ++c) tma_load_2d(tmB, bar, sb + c * 8192, n0 + c * 64, kb * 64);
  }
}

template <int BN, bool SM>
__global__ void __launch_bounds__(256, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
  using Cfg = GemmCfg<BN, SM>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int total = args.units;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    fence_barrier_init();
  }
  __syncthreads();  // barriers initialised
  // PDL: barrier init / descriptor prefetch above overlap the previous kernel; the successor
  // may start its own prologue (it takes TMEM only after its griddepcontrol.wait, i.e. after
  // this grid has completed)
  griddep_launch();
  // weights do not depend on the previous kernel: the first tile's B stages are in flight
  // before griddepcontrol.wait (the weight-stream fill overlaps the predecessor's tail)
  int pre = 0;
  if (warp == 0 && lane == 0 && args.b_const && (int)blockIdx.x < total) {
    int mb, nb, kb0, kb1;
    decode_work(blockIdx.x, args, mb, nb, kb0, kb1);
    pre = min(Cfg::STAGES, kb1 - kb0);
    for (int i = 0; i < pre; ++i) {
      mbar_arrive_expect_tx(&full_bar[i], Cfg::STAGE_BYTES);
      load_b<BN>(&tmB, &full_bar[i], smem + i * Cfg::STAGE_BYTES + Cfg::A_BYTES, kb0 + i, nb * BN,
                 args.b_mn);
    }
  }
  griddep_wait();
  // TMEM only after griddepcontrol.wait: TMEM is an SM-wide resource, and a grid that held it
  // while waiting on an unfinished predecessor could starve that predecessor's not-yet-allocated
  // CTAs on the same SM (a timing-dependent deadlock)
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool first = true;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        int mb, nb, kb0, kb1;
        decode_work(w, args, mb, nb, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (first && kb - kb0 < pre) {  // B already issued for this stage
            tma_load_2d(&tmA, &full_bar[stage], sa, kb * Cfg::BK, mb * Cfg::BM);
          } else {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
            tma_load_2d(&tmA, &full_bar[stage], sa, kb * Cfg::BK, mb * Cfg::BM);
            load_b<BN>(&tmB, &full_bar[stage], sb, kb, nb * BN, args.b_mn);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        first = false;
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the schedule (descriptors stay in uniform registers: no per-MMA
    // R2UR / elect loop), one elected lane issues
    {
      const uint32_t idesc = args.b_mn ? idesc_bf16_f32_major(128, BN, 0, 1) : idesc_bf16_f32(128, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        int mb, nb, kb0, kb1;
        decode_work(w, args, mb, nb, kb0, kb1);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
          const uint64_t ad = umma_desc_sw128(sa);
          const uint64_t bd = umma_desc_sw128(sb);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < Cfg::BK / 16; ++k) {
              // K-major: +32 bytes per K=16 step inside the 128B swizzle atom (16-byte units);
              // MN-major: +16 rows x 128 B, 64-column chunks 8 KB apart (LBO), 8-row groups (SBO)
              const uint64_t b = args.b_mn ? umma_desc_sw128_mn(sb + k * 2048, 8192, 1024)
                                           : bd + (uint64_t)(k * 2);
              mma_bf16(d_tmem, ad + (uint64_t)(k * 2), b, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            mma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) mma_commit(&tfull_bar[acc]);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;  // == warp % 4 -> TMEM lanes [32*ew, 32*ew+32)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      int mb, nb, kb0, kb1;
      decode_work(w, args, mb, nb, kb0, kb1);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * Cfg::BM + ew * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      if constexpr (BN >= 128) {
        if (args.epi == EPI_QKV_ROPE) {
          long prow;
          int pos;
          qkv_row_slot(args, row, prow, pos);
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 128) epilogue_qkv_rope(args, row, nb * BN + c0, tbase + c0, prow, pos);
          tc_fence_before();
          mbar_arrive(&tempty_bar[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
          continue;
        }
        if (args.epi == EPI_SWIGLU) {
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 128)
#pragma unroll 1
            for (int h = 0; h < 64; h += 32) {
              uint32_t g[32], u[32];
              tmem_ld_32x32b_x32(tbase + c0 + h, g);
              tmem_ld_32x32b_x32(tbase + c0 + 64 + h, u);
              tmem_ld_wait();
              epilogue_swiglu(args, row, nb * BN + c0 + h, g, u);
            }
          tc_fence_before();
          mbar_arrive(&tempty_bar[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
          continue;
        }
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += Cfg::CHUNK) {
        const int col0 = nb * BN + c0;
        uint32_t r[32];
        if constexpr (Cfg::CHUNK == 32) {
          tmem_ld_32x32b_x32(tbase + c0, r);
        } else {
          uint32_t r16[16];
          tmem_ld_32x32b_x16(tbase + c0, r16);
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = r16[i];
        }
        tmem_ld_wait();
        if (col0 < args.N) epilogue_store<BN>(args, row, col0, r, Cfg::CHUNK);
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ 2-SM (CTA pair) variant
// cta_group::2: a cluster of 2 CTAs on one TPC computes a 256 x BN tile; CTA r loads A rows
// [128r, 128r+128) and B rows [BN/2 r, BN/2 r + BN/2) of the tile into its own shared memory,
// the leader (rank 0) issues tcgen05.mma.cta_group::2 (M=256), and each CTA's TMEM receives
// its 128 accumulator rows x BN.  Per SM that halves the B-operand shared-memory traffic of
// the 1-SM kernel (the tensor pipe stalls on operand delivery at M=128, N=256).
//   full[s]   (leader)     : leader arrive.expect_tx(both CTAs' bytes); both CTAs' TMA
//                            complete_tx on it (2-SM TMA form, peer bit cleared)
//   empty[s]  (each CTA)   : leader's MMA commit, multicast to both CTAs
//   tfull[a]  (each CTA)   : leader's accumulator commit, multicast
//   tempty[a] (leader)     : 256 arrivals, the peer's epilogue arrives remotely (mapa)
template <int BN>
struct Gemm2Cfg {
  static constexpr int BK = 64;
  static constexpr int A_BYTES = 128 * BK * 2;        // this CTA's 128 rows of A
  static constexpr int B_BYTES = (BN / 2) * BK * 2;   // this CTA's half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES > 8 ? 8 : (192 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

namespace {
CS_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
CS_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-SM TMA load: data into this CTA's smem, transaction bytes to the leader CTA's mbarrier
CS_DEV void tma_load_2d_2sm(const CUtensorMap* m, uint64_t* bar, void* smem, int c0, int c1) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(b), "r"(c0), "r"(c1)
      : "memory");
}
CS_DEV void mma_bf16_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
CS_DEV void mma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)0x3)
      : "memory");
}
// arrive on the leader CTA's copy of `bar`
CS_DEV void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// this CTA's half of a B stage (BN/2 columns x 64 K), 2-SM TMA
template <int BN>
CS_DEV void load_b_2sm(const CUtensorMap* tmB, uint64_t* bar, uint8_t* sb, int kb, int n0, int b_mn) {
  if (!b_mn) {
    tma_load_2d_2sm(tmB, bar, sb, kb * 64, n0);
  } else {
#pragma unroll
    for (int c = 0; c < BN / 128; ++c) tma_load_2d_2sm(tmB, bar, sb + c * 8192, n0 + c * 64, kb * 64);
  }
}
}  // namespace

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_tn2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmArgs args) {
  using Cfg = Gemm2Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull_bar = empty_bar + Cfg::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);  // warp-uniform
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int total = args.units;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 256);
    }
    fence_barrier_init();
  }
  cluster_sync_all();  // barriers initialised in both CTAs (the peer's TMA signals the leader's)
  griddep_launch();
  int pre = 0;  // first tile's B (weight) stages issued before griddepcontrol.wait
  if (warp == 0 && lane == 0 && args.b_const && pair < total) {
    int mb, nb, kb0, kb1;
    decode_work(pair, args, mb, nb, kb0, kb1);
    pre = min(Cfg::STAGES, kb1 - kb0);
    for (int i = 0; i < pre; ++i) {
      if (leader) mbar_arrive_expect_tx(&full_bar[i], 2 * Cfg::STAGE_BYTES);
      load_b_2sm<BN>(&tmB, &full_bar[i], smem + i * Cfg::STAGE_BYTES + Cfg::A_BYTES, kb0 + i,
                     nb * BN + (int)rank * (BN / 2), args.b_mn);
    }
  }
  griddep_wait();
  // TMEM only after griddepcontrol.wait (see gemm_tn_kernel)
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool first = true;
      for (int w = pair; w < total; w += n_pairs) {
        int mb, nb, kb0, kb1;
        decode_work(w, args, mb, nb, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (first && kb - kb0 < pre) {
            tma_load_2d_2sm(&tmA, &full_bar[stage], sa, kb * Cfg::BK, mb * 256 + (int)rank * 128);
          } else {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
            tma_load_2d_2sm(&tmA, &full_bar[stage], sa, kb * Cfg::BK, mb * 256 + (int)rank * 128);
            load_b_2sm<BN>(&tmB, &full_bar[stage], sb, kb, nb * BN + (int)rank * (BN / 2), args.b_mn);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        first = false;
      }
    }
  } else if (warp == 1) {
    // leader CTA: the whole warp walks the schedule (uniform descriptors), one lane issues
    if (leader) {
      const uint32_t idesc = args.b_mn ? idesc_bf16_f32_major(256, BN, 0, 1) : idesc_bf16_f32(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = pair; w < total; w += n_pairs) {
        int mb, nb, kb0, kb1;
        decode_work(w, args, mb, nb, kb0, kb1);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
          const uint64_t ad = umma_desc_sw128(sa);
          const uint64_t bd = umma_desc_sw128(sb);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < Cfg::BK / 16; ++k) {
              const uint64_t b = args.b_mn ? umma_desc_sw128_mn(sb + k * 2048, 8192, 1024)
                                           : bd + (uint64_t)(k * 2);
              mma_bf16_2sm(d_tmem, ad + (uint64_t)(k * 2), b, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            mma_commit_2sm(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) mma_commit_2sm(&tfull_bar[acc]);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = pair; w < total; w += n_pairs) {
      int mb, nb, kb0, kb1;
      decode_work(w, args, mb, nb, kb0, kb1);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * 256 + (int)rank * 128 + ew * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      if (args.epi == EPI_QKV_ROPE) {
        long prow;
        int pos;
        qkv_row_slot(args, row, prow, pos);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 128) epilogue_qkv_rope(args, row, nb * BN + c0, tbase + c0, prow, pos);
      } else if (args.epi == EPI_SWIGLU) {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 128)
#pragma unroll 1
          for (int h = 0; h < 64; h += 32) {
            uint32_t g[32], u[32];
            tmem_ld_32x32b_x32(tbase + c0 + h, g);
            tmem_ld_32x32b_x32(tbase + c0 + 64 + h, u);
            tmem_ld_wait();
            epilogue_swiglu(args, row, nb * BN + c0 + h, g, u);
          }
      } else {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          const int col0 = nb * BN + c0;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + c0, r);
          tmem_ld_wait();
          if (col0 < args.N) epilogue_store<BN>(args, row, col0, r, 32);
        }
      }
      tc_fence_before();
      mbar_arrive_leader(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // every MMA into / operand read from both CTAs has completed
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)Cfg::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  long rows, cols, ld;
  int box_rows;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld &&
           box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.ptr);
    h ^= (size_t)k.rows * 0x9E3779B97F4A7C15ull + (size_t)k.cols * 31 + (size_t)k.ld * 131 +
         (size_t)k.box_rows * 7;
    return h;
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

}  // namespace

int make_map(CUtensorMap* out, const void* ptr, long rows, long cols, long ld, int box_rows) {
  MapKey key{ptr, rows, cols, ld, box_rows};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return 0;
    }
  }
  auto enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -2;
  std::lock_guard<std::mutex> lk(g_map_mu);
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = *out;
  return 0;
}

// 3D bf16 map (dims innermost first), SWIZZLE_128B, box = {64, box1, box2}; strides in bytes
int make_map_3d(CUtensorMap* out, const void* ptr, long d0, long d1, long d2, long stride1_bytes,
                long stride2_bytes, int box1, int box2) {
  auto enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)stride1_bytes, (cuuint64_t)stride2_bytes};
  cuuint32_t box[3] = {64, (cuuint32_t)box1, (cuuint32_t)box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// 3D bf16 map without swizzle, box = {box0, box1, box2} (dims innermost first, strides in
// bytes): the canonical no-swizzle UMMA layouts, e.g. 8-element (16-byte) core-matrix rows
int make_map_3d_plain(CUtensorMap* out, const void* ptr, long d0, long d1, long d2, long stride1_bytes,
                      long stride2_bytes, int box0, int box1, int box2) {
  auto enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)stride1_bytes, (cuuint64_t)stride2_bytes};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, (cuuint32_t)box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int make_map_3d_f32(CUtensorMap* out, const void* ptr, long d0, long d1, long d2, long stride1_bytes,
                    long stride2_bytes, int box0, int box1, int box2) {
  auto enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)stride1_bytes, (cuuint64_t)stride2_bytes};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, (cuuint32_t)box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

namespace {

template <int BN, bool SM = false>
cudaError_t launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a,
                      int grid, cudaStream_t st) {
  using Cfg = GemmCfg<BN, SM>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel<BN, SM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  return launch_pdl(gemm_tn_kernel<BN, SM>, dim3(grid), dim3(256), Cfg::SMEM, st, ma, mb, a);
}

}  // namespace

int gemm_pick_bn(long M, long N) {
  const long mt = (M + 127) / 128;
  if (N <= 16) return 16;
  if (N <= 32) return 32;
  // largest BN that still gives ~a full wave of tiles
  for (int bn : {256, 128}) {
    if (mt * ((N + bn - 1) / bn) >= 120) return bn;
  }
  return 64;
}

namespace {
bool use_2sm() {
  static const bool on = [] {
    const char* v = std::getenv("CS_GEMM_2SM");
    return !(v && std::atoi(v) == 0);
  }();
  return on;
}

// 256 x BN tiles on CTA pairs, persistent over the pairs (<= 74 pairs on 148 SMs)
template <int BN>
cudaError_t gemm_tn_2sm(const GemmDesc& d, cudaStream_t st, int k_splits = 1) {
  using Cfg = Gemm2Cfg<BN>;
  GemmArgs a;
  a.M = (int)d.M;
  a.N = (int)d.N;
  a.K = (int)d.K;
  a.kb_total = (int)((d.K + 63) / 64);
  a.num_m = (int)((d.M + 255) / 256);
  a.num_n = (int)((d.N + BN - 1) / BN);
  a.group_m = group_m_for(a.num_m);
  a.epi = d.epi;
  a.C = d.C;
  a.ldc = d.ldc;
  a.bias = d.bias;
  a.b_const = d.b_const;
  a.sc = d.scatter;
  a.splits = 1;
  a.b_mn = d.b_mn;
  a.C2 = d.C2;
  a.ldc2 = d.ldc2;
  a.c2_row0 = d.c2_row0;
  a.m_cols = (int)(d.N / 2);
  a.qkv = d.qkv;
  const long tiles2 = (long)a.num_m * a.num_n;
  a.units = (int)tiles2;
  if (k_splits > 1) {  // fewer tiles than pairs (EPI_F32): uniform K split, atomics into zeroed C
    cudaError_t e = cudaMemset2DAsync(d.C, d.ldc * sizeof(float), 0, d.N * sizeof(float), d.M, st);
    if (e != cudaSuccess) return e;
    a.splits = k_splits;
    a.units = (int)(tiles2 * k_splits);
  }
  // accumulating epilogues (C += acc): split the last, partial wave of tiles along K when the
  // modelled time -- waves x (K blocks per unit + ~14 blocks of fill / epilogue) -- drops
  // (down projection M=1728: 112 tiles = 1.51 waves on 74 pairs)
  static const bool tail_on = [] {
    const char* v = std::getenv("CS_GEMM_TAIL");
    return !(v && std::atoi(v) == 0);
  }();
  const long np = kNumSMs / 2;
  if (k_splits <= 1 && tail_on && (d.epi == EPI_F32_ADD || d.epi == EPI_F32_ATOMIC) && tiles2 > np && tiles2 % np) {
    const long full = tiles2 / np * np, rem = tiles2 - full;
    const double kb = a.kb_total;
    double best = (double)(full / np + 1) * (kb + 14.0);
    int best_s = 1;
    for (int sp = 2; sp <= 8 && kb / sp >= 8; ++sp) {
      const double c = (double)(full / np) * (kb + 14.0) + (double)((rem * sp + np - 1) / np) * (kb / sp + 14.0);
      if (c < best - 1e-9) best = c, best_s = sp;
    }
    if (best_s > 1) {
      a.full_units = (int)full;
      a.splits = best_s;
      a.units = (int)(full + rem * best_s);
    }
  }
  CUtensorMap ma, mb;
  const long a_rows = d.a_rows > 0 ? d.a_rows : d.M;
  const long b_rows = d.b_rows > 0 ? d.b_rows : d.N;
  if (make_map(&ma, d.A, a_rows, d.K, d.lda, 128) != 0) return cudaErrorInvalidValue;
  if (d.b_mn ? make_map(&mb, d.B, d.K, d.N, d.ldb, 64) != 0
             : make_map(&mb, d.B, b_rows, d.K, d.ldb, BN / 2) != 0)
    return cudaErrorInvalidValue;
  const long work = a.units;
  const int pairs = (int)std::min<long>(work, kNumSMs / 2);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  return launch_pdl(gemm_tn2_kernel<BN>, dim3(2 * pairs), dim3(256), Cfg::SMEM, st, ma, mb, a);
}
}  // namespace

cudaError_t gemm_tn(const GemmDesc& d, cudaStream_t st) {
  if (d.M <= 0 || d.N <= 0) return cudaSuccess;
  static FILE* glog = [] {  // CS_GEMM_LOG=<file>: one line per GEMM (shape census, debugging)
    const char* v = std::getenv("CS_GEMM_LOG");
    return v ? std::fopen(v, "w") : nullptr;
  }();
  if (glog) std::fprintf(glog, "%ld %ld %ld %d\n", d.M, d.N, d.K, d.epi);
  if (d.K <= 0 || (d.K % 8) != 0 || (d.lda % 8) != 0 || (d.ldb % 8) != 0)
    return cudaErrorInvalidValue;
  if (d.epi == EPI_SWIGLU && (d.N % 128 != 0 || (d.m_cols != 0 && d.m_cols * 2 != d.N) || d.ldc < d.N / 2 ||
                              (d.ldc % 8) != 0))
    return cudaErrorInvalidValue;
  if (d.epi == EPI_QKV_ROPE && (d.N % 128 != 0 || d.qkv.q_dim % 128 != 0 || d.qkv.kv_dim % 128 != 0 ||
                                !d.qkv.row_pos || !d.qkv.row_slot || !d.qkv.k_pool || !d.qkv.v_pool || !d.qkv.rope_tab))
    return cudaErrorInvalidValue;
  // bf16-output epilogues: no K split (EPI_SWIGLU / EPI_QKV_ROPE as EPI_BF16 below)
  const bool bf16_out = d.epi == EPI_BF16 || d.epi == EPI_SWIGLU || d.epi == EPI_QKV_ROPE;
  // large GEMMs (at least one wave of 256 x BN tiles): CTA-pair kernel
  if (d.bn <= 0 && d.splits <= 0 && use_2sm() && d.M >= 256) {
    const long mt = (d.M + 255) / 256;
    // (256 x 128 pair tiles measured slower even where they quantise better onto the 74
    // pairs: QKV M=1728 78 -> 108 us, scripts/gemm_cfg_sweep.py)
    if (d.M >= 512 && mt * ((d.N + 255) / 256) >= kNumSMs / 2) return gemm_tn_2sm<256>(d, st);
    // fewer 256 x 256 tiles than pairs but a long K (the LM head's dH = dlogits U, K = V): split K
    // uniformly so the units fill whole waves of pairs -- waves x (k-blocks / split + ~14)
    const long t2 = mt * ((d.N + 255) / 256), kbt = (d.K + 63) / 64;
    if (d.epi == EPI_F32 && d.M >= 512 && t2 >= 16 && kbt >= 512) {
      const int np = kNumSMs / 2;
      int best_s = 1;
      double best = 1e30;
      for (int sp = 2; sp <= 16 && kbt / sp >= 32; ++sp) {
        const double c = (double)((t2 * sp + np - 1) / np) * ((double)kbt / sp + 14.0);
        if (c < best - 1e-9) best = c, best_s = sp;
      }
      if (best_s > 1) return gemm_tn_2sm<256>(d, st, best_s);
    }
    // (256 x 128 pair tiles measured neutral-to-negative in the co-serving bench: not used)
  }
  int bn = d.bn > 0 ? d.bn : gemm_pick_bn(d.M, d.N);
  // small-M fp32-epilogue GEMMs (the O / down projections of inference-only rows): weight
  // streaming is latency-bound per CTA, so wider tiles split along K beat narrow tiles
  // (scripts/gemm_smallm.py: down T=64 38 us at bn 128 x 4 splits vs 51 us at bn 64 x 3)
  // M <= 64 (decode-only rows): half-height A stages (GemmCfg<.., true>), tile width chosen to
  // minimise waves x bytes-per-stage, fp32 epilogues split along K over ~one wave
  static const bool smallm_on = [] {
    const char* v = std::getenv("CS_GEMM_SMALLM");
    return !(v && std::atoi(v) == 0);
  }();
  const bool tiny_m = smallm_on && d.bn <= 0 && d.splits <= 0 && d.M <= 64 && d.N >= 1024;
  if (tiny_m) {
    if (bf16_out) {
      long best = -1;
      for (int c : {256, 128, 64}) {  // >= 64: the MMA's phantom A rows stay inside the stage
        const long waves = (((d.N + c - 1) / c) + kNumSMs - 1) / kNumSMs;
        const long cost = waves * (8192 + (long)c * 128);
        if (best < 0 || cost < best) best = cost, bn = c;
      }
    } else {
      bn = 256;
    }
  }
  const bool small_f32 = !tiny_m && d.bn <= 0 && d.splits <= 0 && !bf16_out && d.M <= 256 &&
                         d.N >= 1024;
  if (small_f32) bn = 128;
  // mid-M fp32 epilogues that missed the CTA-pair kernel (the O / down projections and dX
  // GEMMs of backward-phase iterations, M ~ 500-1100): pick tile width x K splits by waves x
  // per-unit time, a unit = its K blocks + a fixed ~14-block cost (pipeline fill, fp32
  // epilogue; fitted on scripts/gemm_cfg_sweep.py), a BN=128 tile doing half the work of a
  // 256 one at ~85% of its per-FLOP rate.  M=640 N=4096 K=14400: 130 us (bn 128, 1 split,
  // 160 tiles = 1.08 waves) -> 80 us (bn 256 x 3 splits)
  int mid_splits = 0;
  if (!tiny_m && !small_f32 && d.bn <= 0 && d.splits <= 0 && !bf16_out && d.N >= 1024) {
    const long kb = (d.K + 63) / 64;
    double best = 0;
    for (int c : {256, 128}) {
      const long tiles = ((d.M + 127) / 128) * ((d.N + c - 1) / c);
      for (long sp = 1; sp <= 8 && (sp == 1 || kb / sp >= 8); ++sp) {
        const long waves = (tiles * sp + kNumSMs - 1) / kNumSMs;
        const double cost = (double)waves * ((double)kb / (double)sp + 14.0) * c / (c == 256 ? 1.0 : 0.85);
        if (best == 0 || cost < best - 1e-9) best = cost, bn = c, mid_splits = (int)sp;
      }
    }
  }
  if (d.b_mn && bn < 64) bn = 64;  // MN-major B stages are 64-column chunks
  if ((d.epi == EPI_SWIGLU || d.epi == EPI_QKV_ROPE) && bn < 128) bn = 128;  // whole 128-column groups per tile
  GemmArgs a;
  a.M = (int)d.M;
  a.N = (int)d.N;
  a.K = (int)d.K;
  a.kb_total = (int)((d.K + 63) / 64);
  a.num_m = (int)((d.M + 127) / 128);
  a.num_n = (int)((d.N + bn - 1) / bn);
  a.group_m = group_m_for(a.num_m);
  a.epi = d.epi;
  a.C = d.C;
  a.ldc = d.ldc;
  a.bias = d.bias;
  a.b_const = d.b_const;
  a.sc = d.scatter;
  a.C2 = d.C2;
  a.ldc2 = d.ldc2;
  a.c2_row0 = d.c2_row0;
  a.m_cols = (int)(d.N / 2);
  a.qkv = d.qkv;
  int splits = d.splits > 0 ? d.splits : mid_splits;
  const long tiles = (long)a.num_m * a.num_n;
  if (splits <= 0) {
    splits = 1;
    if (tiny_m && !bf16_out) {
      // M <= 64 (half-height A stages, more weight bytes in flight per CTA): ~one unit per SM
      splits = (int)((kNumSMs + tiles / 2) / tiles);
      splits = std::max(1, std::min(splits, a.kb_total / 8));
    } else if (small_f32) {
      // 64 < M <= 256: whole waves, minimise waves x (k-blocks per unit + ~14 blocks of fill /
      // epilogue) -- rounding 148 / tiles to the nearest count gave 5 splits x 32 tiles = 160
      // units, 1.08 waves, for the M = 81 O / down projections: 20.5 / 43.8 -> 18.4 / 36.9 us,
      // a decode-only 8B step with 81 rows 5.42 -> 5.03 ms (scripts/decode_step_bench.py)
      double best = 0;
      for (int sp = 1; sp <= 16 && (sp == 1 || a.kb_total / sp >= 8); ++sp) {
        const double c = (double)((tiles * sp + kNumSMs - 1) / kNumSMs) * ((double)a.kb_total / sp + 14.0);
        if (best == 0 || c < best - 1e-9) best = c, splits = sp;
      }
    } else if (!bf16_out && tiles < kNumSMs) {
      // fewer tiles than SMs (the LoRA products, N = r = 16): whole waves as above -- the ceil
      // gave 10 splits x 16 tiles = 160 units for u = m A at 2K rows
      double best = 0;
      for (int sp = 1; sp <= 64 && (sp == 1 || a.kb_total / sp >= 4); ++sp) {
        const double c = (double)((tiles * sp + kNumSMs - 1) / kNumSMs) * ((double)a.kb_total / sp + 14.0);
        if (best == 0 || c < best - 1e-9) best = c, splits = sp;
      }
    }
  }
  if (bf16_out) splits = 1;
  splits = std::max(1, std::min(splits, a.kb_total));
  a.splits = splits;
  a.units = (int)((long)a.num_m * a.num_n * splits);
  if (d.epi == EPI_F32 && splits > 1) {
    cudaError_t e = cudaMemset2DAsync(d.C, d.ldc * sizeof(float), 0, d.N * sizeof(float), d.M, st);
    if (e != cudaSuccess) return e;
  }
  a.b_mn = d.b_mn;
  CUtensorMap ma, mb;
  const long a_rows = d.a_rows > 0 ? d.a_rows : d.M;
  const long b_rows = d.b_rows > 0 ? d.b_rows : d.N;
  if (make_map(&ma, d.A, a_rows, d.K, d.lda, tiny_m ? 64 : 128) != 0) return cudaErrorInvalidValue;
  if (d.b_mn ? make_map(&mb, d.B, d.K, d.N, d.ldb, 64) != 0 : make_map(&mb, d.B, b_rows, d.K, d.ldb, bn) != 0)
    return cudaErrorInvalidValue;
  const long work = tiles * splits;
  const int grid = (int)std::min<long>(work, d.max_ctas > 0 ? d.max_ctas : kNumSMs);
  if (tiny_m) {
    switch (bn) {
      case 64: return launch_bn<64, true>(ma, mb, a, grid, st);
      case 128: return launch_bn<128, true>(ma, mb, a, grid, st);
      case 256: return launch_bn<256, true>(ma, mb, a, grid, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (bn) {
    case 16: return launch_bn<16>(ma, mb, a, grid, st);
    case 32: return launch_bn<32>(ma, mb, a, grid, st);
    case 64: return launch_bn<64>(ma, mb, a, grid, st);
    case 128: return launch_bn<128>(ma, mb, a, grid, st);
    case 256: return launch_bn<256>(ma, mb, a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cs
