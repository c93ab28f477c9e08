// attn_bwd2.cu -- K9: the attention part of a token-level backward window (Alg. 2 lines 14-21,
// PAPER.md:353-364; tiny_model.hpp:294-315 for query rows [a, b) over keys [0, b)) as ONE tcgen05
// kernel per window: dK / dV accumulate in TMEM per 128-key block, dQ is reduce-added into fp32
// per (key block, query tile).  P is recomputed from Q, K and the saved LSE; exp2 on the SFU
// (ex2.approx), the rest on FFMA2 / FADD2 / FMUL2.  Design and measurements: DESIGN.md §4 (K9).
#include <atomic>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"

namespace cs {

// ---- in-kernel event trace (debugging): SM-clock timeline of one CTA (key block == cta,
// kv head 0) of the backward kernels, set by cs_debug_trace(); compiled in only for the
// trace build (python -m paper_2402_18789_b200.build --trace -> libcoserve_cuda_trace.so): the
// check reads a __device__ global, a load on the MMA issuer's critical path
__device__ int g_trace_cta = -1;
__device__ unsigned long long* g_trace_buf = nullptr;
__device__ __forceinline__ void trace_ev(int ev, int idx) {
#if !defined(CS_TRACE) && !defined(CS_TRACE_CHECK)
  (void)ev;
  (void)idx;
  return;
#endif
  if ((int)blockIdx.y != g_trace_cta || blockIdx.x != 0) return;
  // one slot per (event, index): a plain store, no atomic round trip on the traced path
  if (idx < 4096 && ev < 64) {
    unsigned long long* slot = g_trace_buf + ev * 4096 + idx;
    if (ev == 35 || ev == 36) {  // "first seen" events: keep the earliest
      if (*slot == 0) *slot = clock64();
    } else {
      *slot = clock64();
    }
  }
}

namespace {
constexpr float kLog2eC = 1.4426950408889634f;
constexpr int DB = 128;
constexpr int HALFB = 128 * 128;  // [128 rows][128 B] = 16 KB
constexpr int TILEB = 2 * HALFB;  // 32 KB


CS_DEV void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

CS_DEV void tst_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

CS_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }


// paged K and V tile of 128 keys -> two SW128 halves each (contiguous-run fast path)
CS_DEV void load_kv2(const CUtensorMap* tK, const CUtensorMap* tV, const CUtensorMap* tK128,
                     const CUtensorMap* tV128, uint64_t* bar, uint8_t* sk, uint8_t* sv, const int* pt,
                     int page_off, int P, int k0, int k_end, int kvh) {
  const int pg0 = __ldg(pt + page_off + k0 / P);
  bool contig = true;
  for (int key = (k0 / P + 1) * P; key < k0 + 128 && key < k_end; key += P)
    contig &= __ldg(pt + page_off + key / P) == pg0 + (key / P - k0 / P);
  if (contig) {
    const int row = pg0 * P + (k0 % P);
    for (int h = 0; h < 2; ++h) {
      tma_load_2d(tK128, bar, sk + h * HALFB, kvh * DB + h * 64, row);
      tma_load_2d(tV128, bar, sv + h * HALFB, kvh * DB + h * 64, row);
    }
  } else {
    for (int ch = 0; ch < 8; ++ch) {
      const int key0 = k0 + ch * 16;
      const int row = key0 < k_end ? __ldg(pt + page_off + key0 / P) * P + (key0 % P) : 0;
      for (int h = 0; h < 2; ++h) {
        tma_load_2d(tK, bar, sk + h * HALFB + ch * 2048, kvh * DB + h * 64, row);
        tma_load_2d(tV, bar, sv + h * HALFB + ch * 2048, kvh * DB + h * 64, row);
      }
    }
  }
}
}  // namespace

// ============================================================================ fused dK / dV / dQ
// One pass over (128-key block, 64-row packed query tile) pairs computes all five products:
//   S^T = K Q^T, dP^T = V dO^T                 (M = 128 keys, N = 64 rows: TMEM, single buffer)
//   P^T = exp2(S^T scale_log2 - lse2), dS^T = P^T (dP^T - Delta)   (8 elementwise warps)
//   dV += P^T dO  (A = P^T from TMEM),  dK += dS^T Q  (A = dS^T from SMEM, K-major SW128)
//   dQ^T = K^T dS^T  (M = 128 head dims, N = 64 rows: A = the K tile read MN-major, B = the same
//                     dS^T buffer read MN-major), read out by 4 warps and added into the fp32 dQ
//                     of the window with TMA bulk tensor reduce-add (cp.reduce.async.bulk.tensor)
// -- no dS round trip through HBM (the dS-export design wrote and re-read 2 B per (key, row)
// pair) and no S / dP recompute for dQ.  The S^T / dP^T TMEM buffer is released as soon as the
// elementwise warps hold it in registers, so S^T(i+1) / dP^T(i+1) run on the tensor pipe while
// they compute tile i, and dV / dK / dQ^T of tile i run while they compute tile i+1.
// MMA issue is warp-uniform (descriptors in uniform registers): a per-MMA R2UR + elect loop cost
// ~108 clk per N=64 MMA in the dK/dV kernel above, against a 48 clk hardware floor
// (scripts/micro/mma_rate.cu).
namespace kv3 {
constexpr int QB = 64;                  // packed query rows per tile
constexpr int HALFQ = QB * 128;         // 8 KB: one 64-column half of a Q / dO tile
constexpr int QTILE = 2 * HALFQ;        // 16 KB
constexpr int QST = 3;                  // Q / dO ring depth (a stage is held from S^T(i) until dV / dK(i))
constexpr int SMEM_K = 0;
constexpr int SMEM_V = SMEM_K + TILEB;
constexpr int SMEM_Q = SMEM_V + TILEB;
constexpr int SMEM_O = SMEM_Q + QST * QTILE;
constexpr int SMEM_DS = SMEM_O + QST * QTILE;  // dS^T [128 keys][64 rows] bf16, K-major SW128: 16 KB
constexpr int XST = 2;                  // x ring depth
constexpr int SMEM_DQ = SMEM_DS + 128 * 128;   // dQ staging: [2 head-dim halves][64 rows][64] f32
constexpr int SMEM_X = SMEM_DQ + 2 * QB * 64 * 4;  // [XST slots][2][QB] f32: -lse*log2e | -Delta
constexpr int SMEM_BAR = SMEM_X + XST * 2 * QB * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;
// TMEM columns: S^T, dP^T (fp32, 64 rows), P^T, dS^T (bf16 pairs), dQ^T (fp32), dV, dK
constexpr uint32_t TM_S = 0, TM_DP = 64, TM_P = 128, TM_DS = 160, TM_DQ = 192, TM_DV = 256, TM_DK = 384;
}  // namespace kv3

template <int GRP>
__global__ void __launch_bounds__(512, 1)
    attn_bwd_fused_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmK128,
                          const __grid_constant__ CUtensorMap tmV128,
                          const __grid_constant__ CUtensorMap tmQ3,
                          const __grid_constant__ CUtensorMap tmO3,
                          const __grid_constant__ CUtensorMap tmDQ, AttnBwdParams p) {
  griddep_launch();  // PDL: a dependent kernel may start its prologue now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  using namespace kv3;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB alignment by pointer arithmetic on the __shared__ array, so the compiler keeps the
  // shared address space (an integer round trip turns every access into a generic LD.E / ST.E)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;             // [QST]
  uint64_t* q_empty = q_full + QST;        // [QST]
  uint64_t* x_full = q_empty + QST;        // [XST] 32 arrivals (loader warp)
  uint64_t* x_empty = x_full + XST;        // [XST] 8 arrivals (one per elementwise warp)
  uint64_t* sd_full = x_empty + XST;       // S^T / dP^T of a tile in TMEM
  uint64_t* sd_free = sd_full + 1;         // 256 arrivals: S^T / dP^T in registers
  uint64_t* pds_full = sd_free + 1;        // 256 arrivals: P^T (TMEM) and dS^T (SMEM) written
  uint64_t* pds_free = pds_full + 1;       // dV / dK / dQ^T MMAs of a tile done
  uint64_t* dq_full = pds_free + 1;        // dQ^T of a tile in TMEM
  uint64_t* dq_free = dq_full + 1;         // 128 arrivals: dQ^T in registers
  uint64_t* acc_done = dq_free + 1;        // all dV / dK MMAs done (completes once)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  constexpr int grp = GRP;
  constexpr int rpt = QB / GRP;            // positions per query tile
  constexpr int ROWS = rpt * GRP;          // real packed rows per tile (<= QB)
  // grid (kv heads, key blocks, splits): the block scheduler's linear order then starts the
  // longest key blocks (the first, causal) of every head first -- LPT over the SMs
  const int k0 = blockIdx.y * 128;
  const int kvh = blockIdx.x;
  const int nrows = p.b - p.a;
  const int n_qt = (nrows + rpt - 1) / rpt;
  // first tile whose last position >= k0; long key blocks are split over gridDim.z CTAs of at
  // most p.tiles_per_cta query tiles each (their ΔKV partial sums then add atomically)
  const int qt_first = k0 > p.a ? (k0 - p.a) / rpt : 0;
  const int qt0 = qt_first + (int)blockIdx.z * p.tiles_per_cta;
  const int n = max(0, min(n_qt - qt0, p.tiles_per_cta));
  const bool split = gridDim.z > 1;
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);  // warp-uniform
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ3);
    tma_prefetch_desc(&tmO3);
    mbar_init(kv_full, 1);
    for (int i = 0; i < QST; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < XST; ++i) {
      mbar_init(&x_full[i], 32);
      mbar_init(&x_empty[i], 8);
    }
    mbar_init(sd_full, 1);
    mbar_init(sd_free, 256);
    mbar_init(pds_full, 256);
    mbar_init(pds_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 128);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if constexpr (ROWS < QB) {  // pad rows [ROWS, QB) of every Q / dO stage, both 128-B halves
    constexpr int PADB = (QB - ROWS) * 128;
    for (int i = threadIdx.x; i < 2 * QST * 2 * (PADB / 16); i += blockDim.x) {
      const int half = i / (PADB / 16), o = (i % (PADB / 16)) * 16;  // half: (Q|O, stage, h)
      *reinterpret_cast<uint4*>(smem + SMEM_Q + half * HALFQ + ROWS * 128 + o) = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  float* xring = reinterpret_cast<float*>(smem + SMEM_X);

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0) {  // TMA producer: K / V once, then the Q / dO ring
      if (lane == 0) {
        if (n > 0) {
          mbar_arrive_expect_tx(kv_full, 2 * TILEB);
          load_kv2(&tmK, &tmV, &tmK128, &tmV128, kv_full, smem + SMEM_K, smem + SMEM_V, p.page_table,
                   p.page_off, p.page_size, k0, p.b, kvh);
        }
        for (int i = 0; i < n; ++i) {
          const int st = i % QST;
          const int qt = qt0 + i;
          mbar_wait(&q_empty[st], ((i / QST) & 1) ^ 1);
          trace_ev(34, i);
          mbar_arrive_expect_tx(&q_full[st], 2 * 2 * ROWS * 128);
          for (int h = 0; h < 2; ++h) {
            tma_load_3d(&tmQ3, &q_full[st], smem + SMEM_Q + st * QTILE + h * HALFQ, h * 64, kvh * grp,
                        p.a + qt * rpt);
            tma_load_3d(&tmO3, &q_full[st], smem + SMEM_O + st * QTILE + h * HALFQ, h * 64, kvh * grp,
                        qt * rpt);
          }
        }
      }
    } else if (warp == 1 || warp == 2) {
      // two MMA issuers, each blocking on its own stream's barriers (tcgen05.commit tracks the
      // issuing thread's MMAs, so the streams stay independent): warp 1 issues S^T / dP^T(i)
      // (Q / dO of tile i landed, S / dP buffer released by the elementwise warps), warp 2
      // dV / dK / dQ^T(j) (P^T / dS^T of tile j written, dQ^T(j-1) read out).  One issuer
      // polling both streams spent ~1.5 K clk per block on probes and MIO back-pressure, with
      // the tensor pipe idle 43% of the time (scripts/micro/mma_rate.cu: the tile's MMAs alone
      // take 1751 clk against ~3.1 K clk per tile in the kernel)
      constexpr uint32_t idS = idesc_bf16_f32_major(128, QB, 0, 0);
      constexpr uint32_t idG = idesc_bf16_f32_major(128, 128, 0, 1);
      constexpr uint32_t idQ = idesc_bf16_f32_major(128, QB, 1, 1);
      const uint32_t sK = smem_u32(smem + SMEM_K), sV = smem_u32(smem + SMEM_V);
      const uint32_t sDS = smem_u32(smem + SMEM_DS);
      if (n > 0) {
        mbar_wait(kv_full, 0);
        tc_fence_after();
      }
      if (warp == 1) {
        for (int i = 0; i < n; ++i) {
          const int st = i % QST;
          mbar_wait(&q_full[st], (i / QST) & 1);
          trace_ev(32, i);
          if (i > 0) mbar_wait(sd_free, (i - 1) & 1);
          tc_fence_after();
          trace_ev(30, i);
          const uint32_t sQ = smem_u32(smem + SMEM_Q + st * QTILE);
          const uint32_t sO = smem_u32(smem + SMEM_O + st * QTILE);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t ak = (kk >> 2) * HALFB + (kk & 3) * 32;
              const uint32_t bq = (kk >> 2) * HALFQ + (kk & 3) * 32;
              mma_bf16(tmem + TM_S, umma_desc_sw128(sK + ak), umma_desc_sw128(sQ + bq), idS, kk > 0);
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t ak = (kk >> 2) * HALFB + (kk & 3) * 32;
              const uint32_t bq = (kk >> 2) * HALFQ + (kk & 3) * 32;
              mma_bf16(tmem + TM_DP, umma_desc_sw128(sV + ak), umma_desc_sw128(sO + bq), idS, kk > 0);
            }
            mma_commit(sd_full);
          }
          __syncwarp();
        }
      } else {
        for (int j = 0; j < n; ++j) {
          const int st = j % QST;
          mbar_wait(pds_full, j & 1);
          trace_ev(33, j);
          if (j > 0) mbar_wait(dq_free, (j - 1) & 1);
          tc_fence_after();
          trace_ev(31, j);
          const uint32_t sQ = smem_u32(smem + SMEM_Q + st * QTILE);
          const uint32_t sO = smem_u32(smem + SMEM_O + st * QTILE);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < QB / 16; ++kk)  // dV += P^T dO   (A = P^T from TMEM)
              mma_ts(tmem + TM_DV, tmem + TM_P + kk * 8, umma_desc_sw128_mn(sO + kk * 2048, HALFQ, 1024), idG,
                     (j > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < QB / 16; ++kk)  // dK += dS^T Q  (A = dS^T from TMEM)
              mma_ts(tmem + TM_DK, tmem + TM_DS + kk * 8, umma_desc_sw128_mn(sQ + kk * 2048, HALFQ, 1024), idG,
                     (j > 0 || kk > 0) ? 1u : 0u);
            mma_commit(&q_empty[st]);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // dQ^T = K^T dS^T  (both operands read MN-major)
              mma_bf16(tmem + TM_DQ, umma_desc_sw128_mn(sK + kk * 2048, HALFB, 1024),
                       umma_desc_sw128_mn(sDS + kk * 2048, HALFB, 1024), idQ, kk > 0);
            mma_commit(dq_full);
            mma_commit(pds_free);
          }
          __syncwarp();
        }
        if (n > 0 && elect_one()) mma_commit(acc_done);
      }
    } else if (warp == 3) {  // per-column -lse*log2(e) and -Delta of each tile into the x ring
      for (int i = 0; i < n; ++i) {
        const int slot = i % XST;
        mbar_wait(&x_empty[slot], ((i / XST) & 1) ^ 1);
        float* xs = xring + slot * 2 * QB;
#pragma unroll
        for (int t = lane; t < QB; t += 32) {
          const int qr = (qt0 + i) * rpt + t / grp, g = t % grp;
          float l2 = 0.f, dl = 0.f;
          if (t < ROWS && qr < nrows) {
            l2 = -p.lse[(long)(p.a + qr) * p.lse_ld + kvh * grp + g] * kLog2eC;
            dl = -p.delta[(long)qr * p.delta_ld + kvh * grp + g];
          }
          xs[t] = l2;
          xs[QB + t] = dl;
        }
        mbar_arrive(&x_full[slot]);
      }
    }
  } else if (warp < 12) {  // elementwise: key row r, packed rows [32c, 32c + 32) of each tile
    const int c = (warp - 4) >> 2;
    const int r = (warp & 3) * 32 + lane;
    const int key = k0 + r;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    uint8_t* ds_row = smem + SMEM_DS + (r >> 3) * 1024 + (r & 7) * 128;
    for (int i = 0; i < n; ++i) {
      const int qbase = (qt0 + i) * rpt;
      mbar_wait(sd_full, i & 1);
      tc_fence_after();
      if (lane == 0 && warp == 4) trace_ev(40, i);
      uint32_t sv[32], dv[32];
      tmem_ld_32x32b_x32(tmem + lane_base + TM_S + c * 32, sv);
      tmem_ld_32x32b_x32(tmem + lane_base + TM_DP + c * 32, dv);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(sd_free);
      mbar_wait(&x_full[i % XST], (i / XST) & 1);
      if (lane == 0 && warp == 4) trace_ev(41, i);
      // valid columns of this half form one range [lo, hi): causal (row position >= key), rows
      // inside the window and the tile, key inside [0, b)
      const int lo = key < p.b ? max(0, grp * (key - p.a - qbase)) - c * 32 : 32;
      const int hi = min(ROWS, grp * (nrows - qbase)) - c * 32;
      const float4* x4 = reinterpret_cast<const float4*>(xring + (i % XST) * 2 * QB + c * 32);
      uint32_t pp[16], pd[16];
      auto body = [&](auto masked) {
#pragma unroll
        for (int cc = 0; cc < 32; cc += 2) {
          const float4 xl4 = x4[cc >> 2], xd4 = x4[QB / 4 + (cc >> 2)];
          const float2 xl = (cc & 2) ? make_float2(xl4.z, xl4.w) : make_float2(xl4.x, xl4.y);
          const float2 xd = (cc & 2) ? make_float2(xd4.z, xd4.w) : make_float2(xd4.x, xd4.y);
          const float2 x = ffma2(make_float2(__uint_as_float(sv[cc]), __uint_as_float(sv[cc + 1])), sc2, xl);
          float2 pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
          if constexpr (decltype(masked)::value) {
            if (cc < lo || cc >= hi) pv.x = 0.f;
            if (cc + 1 < lo || cc + 1 >= hi) pv.y = 0.f;
          }
          const float2 dd = fadd2(make_float2(__uint_as_float(dv[cc]), __uint_as_float(dv[cc + 1])), xd);
          const float2 ds = fmul2(pv, dd);
          pp[cc >> 1] = pack_bf16(pv.x, pv.y);
          pd[cc >> 1] = pack_bf16(ds.x, ds.y);
        }
      };
      if (lo <= 0 && hi >= 32) body(std::false_type{});
      else body(std::true_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(&x_empty[i % XST]);
      if (i > 0) mbar_wait(pds_free, (i - 1) & 1);  // dV / dK / dQ^T of tile i-1 consumed the buffers
      if (lane == 0 && warp == 4) trace_ev(43, i);
      tc_fence_after();
      tst_x16(tmem + lane_base + TM_P + c * 16, pp);
      tst_x16(tmem + lane_base + TM_DS + c * 16, pd);
#pragma unroll
      for (int v = 0; v < 4; ++v) {  // 16-byte chunk 4c + v of this key's 128-byte dS^T row
        const int ch = 4 * c + v;
        *reinterpret_cast<uint4*>(ds_row + ((ch ^ (r & 7)) << 4)) =
            make_uint4(pd[4 * v], pd[4 * v + 1], pd[4 * v + 2], pd[4 * v + 3]);
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      if (lane == 0 && warp == 4) trace_ev(42, i);
      mbar_arrive(pds_full);
    }
    // ΔKVAccum rows [k0, k0+128) of this head: warps of half c own dV / dK columns [64c, 64c + 64)
    if (n > 0) {
      mbar_wait(acc_done, 0);
      tc_fence_after();
      uint32_t a0[32], a1[32];
      tmem_ld_32x32b_x32(tmem + lane_base + TM_DV + c * 64, a0);
      tmem_ld_32x32b_x32(tmem + lane_base + TM_DV + c * 64 + 32, a1);
      tmem_ld_wait();
      // += into ΔKVAccum: plain read-modify-write, or float4 atomics when the key block is split
      auto acc4 = [&](float* dst, const uint32_t* v, float sc) {
#pragma unroll
        for (int t = 0; t < 32; t += 4) {
          const float4 d = make_float4(__uint_as_float(v[t]) * sc, __uint_as_float(v[t + 1]) * sc,
                                       __uint_as_float(v[t + 2]) * sc, __uint_as_float(v[t + 3]) * sc);
          float4* q4 = reinterpret_cast<float4*>(dst + t);
          if (split) {
            atomicAdd(q4, d);
          } else {
            float4 x = *q4;
            x.x += d.x; x.y += d.y; x.z += d.z; x.w += d.w;
            *q4 = x;
          }
        }
      };
      if (key < p.b) {
        float* av = p.dv_acc + (long)key * p.acc_ld + kvh * DB + c * 64;
        acc4(av, a0, 1.f);
        acc4(av + 32, a1, 1.f);
      }
      tmem_ld_32x32b_x32(tmem + lane_base + TM_DK + c * 64, a0);
      tmem_ld_32x32b_x32(tmem + lane_base + TM_DK + c * 64 + 32, a1);
      tmem_ld_wait();
      if (key < p.b) {
        float* ak = p.dk_acc + (long)key * p.acc_ld + kvh * DB + c * 64;
        acc4(ak, a0, p.scale);
        acc4(ak + 32, a1, p.scale);
      }
    }
    tc_fence_before();
  } else {  // dQ read-out: head dims [32q, 32q + 32) (TMEM lanes) x the tile's 64 rows (columns)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;");
    // staged per 64-wide head-dim half ([rows][64] fp32, the TMA box layout) and added into the
    // fp32 dQ with one bulk tensor reduce-add per half: 1.95 ms per 8K window vs 3.7 ms with
    // per-row warp red.global.add of the same values (scripts/attn_bwd_bench.py)
    const int q = warp & 3, half = q >> 1, dl = (q & 1) * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float* stage = reinterpret_cast<float*>(smem + SMEM_DQ) + half * QB * 64;
    const bool issuer = (q & 1) == 0 && lane == 0;
    for (int j = 0; j < n; ++j) {
      mbar_wait(dq_full, j & 1);
      tc_fence_after();
      if (warp == 12 && lane == 0) trace_ev(50, j);
      uint32_t v[64];
      tmem_ld_32x32b_x32(tmem + lane_base + TM_DQ, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld_32x32b_x32(tmem + lane_base + TM_DQ + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(dq_free);
      if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      named_bar(2 + half, 64);  // the previous reduce has read this half's staging buffer
#pragma unroll
      for (int t = 0; t < ROWS; ++t) stage[t * 64 + dl] = __uint_as_float(v[t]) * p.scale;
      fence_proxy_async_smem();
      named_bar(2 + half, 64);
      if (issuer) {
        asm volatile(
            "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                reinterpret_cast<uint64_t>(&tmDQ)),
            "r"(smem_u32(stage)), "r"(half * 64), "r"(kvh * grp), "r"((qt0 + j) * rpt)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

using FusedFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                         const CUtensorMap, const CUtensorMap, const CUtensorMap, AttnBwdParams);
static const FusedFn kFused[8] = {attn_bwd_fused_kernel<1>, attn_bwd_fused_kernel<2>,
                                  attn_bwd_fused_kernel<3>, attn_bwd_fused_kernel<4>,
                                  attn_bwd_fused_kernel<5>, attn_bwd_fused_kernel<6>,
                                  attn_bwd_fused_kernel<7>, attn_bwd_fused_kernel<8>};

cudaError_t attn_bwd_fused(const AttnBwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                           const CUtensorMap& tmK128, const CUtensorMap& tmV128, const CUtensorMap& tmQ3,
                           const CUtensorMap& tmO3, const CUtensorMap& tmDQ, int n_heads, cudaStream_t st) {
  const int rows = p.b - p.a;
  if (rows <= 0) return cudaSuccess;
  if (p.grp < 1 || p.grp > 8) return cudaErrorInvalidValue;
  static bool once = [] {
    for (auto k : kFused)
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kv3::SMEM_TOTAL);
    return true;
  }();
  (void)once;
  // dQ of the window accumulates by reduce-add: zero it first
  cudaError_t err = cudaMemsetAsync(p.dq, 0, (size_t)rows * p.dq_ld * sizeof(float), st);
  if (err != cudaSuccess) return err;
  g_launches.fetch_add(2, std::memory_order_relaxed);
  attn_bwd_delta_kernel_launch(p, rows, n_heads, st);
  // query tiles per key block: n(x) = n_qt - first tile at or after key block x.  A small causal
  // window leaves fewer key-block CTAs than SMs with a 16x spread of lengths (s = 2048 at
  // l_j = 2048: 128 CTAs of 8..128 tiles), so long blocks are split into CTAs of at most
  // ~total / (2 x 148) tiles (>= 24: K / V load and ΔKV epilogue per CTA), spread over grid.z
  const int rpt = 64 / p.grp, nkb = (p.b + 127) / 128, kvh = n_heads / p.grp;
  const long n_qt = (rows + rpt - 1) / rpt;
  long total = 0;
  for (int x = 0; x < nkb; ++x) total += n_qt - (x * 128 > p.a ? (x * 128 - p.a) / rpt : 0);
  total *= kvh;
  AttnBwdParams q = p;
  q.tiles_per_cta = (int)std::max<long>(24, (total + 2 * kNumSMs - 1) / (2 * kNumSMs));
  const int nz = (int)std::min<long>(8, (n_qt + q.tiles_per_cta - 1) / q.tiles_per_cta);
  if ((n_qt + q.tiles_per_cta - 1) / q.tiles_per_cta > 8) q.tiles_per_cta = (int)((n_qt + 7) / 8);
  dim3 grid(kvh, nkb, nz);
  launch_pdl(kFused[p.grp - 1], grid, dim3(512), kv3::SMEM_TOTAL, st, tmK, tmV, tmK128, tmV128, tmQ3, tmO3, tmDQ, q);
  return cudaGetLastError();
}

}  // namespace cs

// trace build only: clock64() of event ev for tile idx of CTA (cta, 0) lands in
// dev_buf[ev * 4096 + idx] (dev_buf: 64 x 4096 int64, zeroed by the caller); cta -1 stops
extern "C" int64_t cs_debug_trace(int cta, void* dev_buf, int64_t capacity) {
  if (capacity < 64 * 4096) return -1;
  cudaMemcpyToSymbol(cs::g_trace_buf, &dev_buf, sizeof(void*));
  cudaMemcpyToSymbol(cs::g_trace_cta, &cta, sizeof(int));
  return 0;
}
