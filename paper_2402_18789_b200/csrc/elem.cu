// elem.cu -- bandwidth-bound kernels of the co-serving step (K4/K5/K6/K11-K14):
// embedding gather (tiny_model.hpp:189-190), RMSNorm / cast, RoPE + paged KV append
// (+ Q-cache append for FT rows), ReLU (tiny_model.hpp:204-205) / SwiGLU,
// LoRA packing for the K-concatenated down projection (tiny_model.hpp:207-211), fused
// cross-entropy forward+backward (row_cross_entropy :170-177, loss_head_grad :223-246),
// token-level backward helpers (tiny_model.hpp:276-319), and the LoRA Adam update.
#include <algorithm>
#include <cfloat>

#include <atomic>

#include "common.cuh"
#include "engine_kernels.h"
#include "kernels.h"

namespace cs {

namespace {

CS_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.f;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  return red[0];
}

CS_DEV float block_max(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float t = (threadIdx.x < nw) ? red[threadIdx.x] : -INFINITY;
  if (w == 0) t = warp_max(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  return red[0];
}

// sigmoid on the SFU (ex2 + rcp.approx; 1/inf -> 0 for x -> -inf): one exp and one reciprocal
// per element instead of two IEEE divisions (the SwiGLU backward was issue-bound on them)
CS_DEV float sigmoid_f(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
CS_DEV float silu_f(float x) { return x * sigmoid_f(x); }
CS_DEV float dsilu_f(float x) {
  const float s = sigmoid_f(x);
  return s * (1.f + x * (1.f - s));
}

}  // namespace

// ---------------------------------------------------------------- embedding
__global__ void embed_kernel(const int* __restrict__ tok, const bf16* __restrict__ E,
                             float* __restrict__ x, int h) {
  const long row = blockIdx.x;
  const bf16* src = E + (long)tok[row] * h;
  float* dst = x + row * h;
  for (int c = threadIdx.x * 8; c < h; c += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(src + c);
    const bf16* b = reinterpret_cast<const bf16*>(&v);
    float4 a0 = make_float4(__bfloat162float(b[0]), __bfloat162float(b[1]),
                            __bfloat162float(b[2]), __bfloat162float(b[3]));
    float4 a1 = make_float4(__bfloat162float(b[4]), __bfloat162float(b[5]),
                            __bfloat162float(b[6]), __bfloat162float(b[7]));
    *reinterpret_cast<float4*>(dst + c) = a0;
    *reinterpret_cast<float4*>(dst + c + 4) = a1;
  }
}
void embed_gather(const int* tokens, const bf16* embed, float* x, int T, int h, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  if (T > 0) embed_kernel<<<T, 128, 0, st>>>(tokens, embed, x, h);
}

// ---------------------------------------------------------------- RMSNorm / cast
// One 128-thread block per row; the row is read once into registers (float4, <= 16 per
// thread: h <= 8192), reduced (shuffles + one smem exchange), scaled and written as bf16.
constexpr int RMS_V = 16;
__global__ void __launch_bounds__(128) rmsnorm_kernel(const float* __restrict__ x, long ldx,
                                                      const int* __restrict__ idx,
                                                      const float* __restrict__ g,
                                                      bf16* __restrict__ out, long ldo,
                                                      float* __restrict__ rstd_out, int h, float eps,
                                                      int use_norm) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  __shared__ float red[4];
  const long src_row = idx ? idx[blockIdx.x] : blockIdx.x;
  const float* xr = x + src_row * ldx;
  bf16* o = out + (long)blockIdx.x * ldo;
  float4 v[RMS_V];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < RMS_V; ++k) {
    const int c = (threadIdx.x + k * 128) * 4;
    v[k] = c < h ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
  }
  float rstd = 1.f;
  if (use_norm) {
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    ss = red[0] + red[1] + red[2] + red[3];
    rstd = rsqrtf(ss / (float)h + eps);
    if (rstd_out && threadIdx.x == 0) rstd_out[blockIdx.x] = rstd;
  }
#pragma unroll
  for (int k = 0; k < RMS_V; ++k) {
    const int c = (threadIdx.x + k * 128) * 4;
    if (c >= h) continue;
    float4 w = v[k];
    if (use_norm) {
      const float4 gg = __ldg(reinterpret_cast<const float4*>(g + c));
      w.x *= rstd * gg.x;
      w.y *= rstd * gg.y;
      w.z *= rstd * gg.z;
      w.w *= rstd * gg.w;
    }
    *reinterpret_cast<uint2*>(o + c) = make_uint2(pack_bf16(w.x, w.y), pack_bf16(w.z, w.w));
  }
}
void rmsnorm_cast(const float* x, long ldx, const float* g, bf16* out, long ldo, float* rstd_out,
                  int rows, int h, float eps, int use_norm, cudaStream_t st) {
  if (rows <= 0) return;
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(rmsnorm_kernel, dim3(rows), dim3(128), 0, st, x, ldx, nullptr, g, out, ldo, rstd_out, h, eps, use_norm);
}
void rmsnorm_cast_gather(const float* x, long ldx, const int* idx, const float* g, bf16* out,
                         long ldo, float* rstd_out, int rows, int h, float eps, int use_norm,
                         cudaStream_t st) {
  if (rows <= 0) return;
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(rmsnorm_kernel, dim3(rows), dim3(128), 0, st, x, ldx, idx, g, out, ldo, rstd_out, h, eps, use_norm);
}

// ---------------------------------------------------------------- RoPE + KV append
__global__ void rope_append_kernel(RopeAppendParams p, const float2* __restrict__ cs_tab) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  const int row = blockIdx.x;
  const int pos = p.row_pos[row];
  const AttnSeg sg = p.segs[p.row_seg[row]];
  const int d = p.head_dim, half = d / 2;
  const int q_dim = p.n_heads * d, kv_dim = p.n_kv_heads * d;
  bf16* q = p.qkv + (long)row * p.ld;
  bf16* k = q + q_dim;
  const bf16* v = k + kv_dim;
  const long prow = (long)__ldg(p.page_table + sg.page_off + pos / p.page_size) * p.page_size +
                    (pos % p.page_size);
  bf16* kd = p.k_pool + prow * kv_dim;
  bf16* vd = p.v_pool + prow * kv_dim;
  const bool ft = row >= p.ft_row0 && p.q_cache;
  bf16* qc = ft ? p.q_cache + (long)pos * q_dim : nullptr;
  const float2* tab = cs_tab + (long)pos * half;
  // q heads (in place) and k heads (to the page): 8 rotate-half pairs (i, i + d/2) per thread,
  // 16-byte loads/stores of both halves
  const int cpr = half / 8;  // 8-pair chunks per head
  const int nq = p.n_heads * cpr, nk = p.n_kv_heads * cpr;
  for (int t = threadIdx.x; t < nq + nk; t += blockDim.x) {
    const bool isq = t < nq;
    const int tt = isq ? t : t - nq;
    const int hd = tt / cpr, i0 = (tt % cpr) * 8;
    bf16* src = (isq ? q : k) + hd * d;
    uint4 a = *reinterpret_cast<const uint4*>(src + i0);
    uint4 b = *reinterpret_cast<const uint4*>(src + i0 + half);
    if (p.use_rope) {
      bf16* xa = reinterpret_cast<bf16*>(&a);
      bf16* xb = reinterpret_cast<bf16*>(&b);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 cs = tab[i0 + j];
        const float x1 = __bfloat162float(xa[j]), x2 = __bfloat162float(xb[j]);
        xa[j] = __float2bfloat16(x1 * cs.x - x2 * cs.y);
        xb[j] = __float2bfloat16(x2 * cs.x + x1 * cs.y);
      }
    }
    if (isq) {
      *reinterpret_cast<uint4*>(src + i0) = a;
      *reinterpret_cast<uint4*>(src + i0 + half) = b;
      if (qc) {
        *reinterpret_cast<uint4*>(qc + hd * d + i0) = a;
        *reinterpret_cast<uint4*>(qc + hd * d + i0 + half) = b;
      }
    } else {
      *reinterpret_cast<uint4*>(kd + hd * d + i0) = a;
      *reinterpret_cast<uint4*>(kd + hd * d + i0 + half) = b;
    }
  }
  for (int c = threadIdx.x * 8; c < kv_dim; c += blockDim.x * 8)
    *reinterpret_cast<uint4*>(vd + c) = *reinterpret_cast<const uint4*>(v + c);
}

static const float2* s_rope_tab = nullptr;
void set_rope_table(const float2* tab) { s_rope_tab = tab; }
void rope_append(const RopeAppendParams& p, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  if (p.T > 0) launch_pdl(rope_append_kernel, dim3(p.T), dim3(128), 0, st, p, s_rope_tab);
}

// ---------------------------------------------------------------- activations
// SwiGLU (silu(g) * u) / ReLU of a gate||up row into m's first f columns, zeros into the
// K-concatenation pad columns [f, ldm).  Thread = ACT_CH chunks of 8 columns 1024 columns apart
// (all loads issued before the math: 4 x 32 B in flight per thread), block = 128 threads.
constexpr int ACT_CH = 4;
__global__ void __launch_bounds__(128) act_kernel(const bf16* __restrict__ gu, long ld_gu,
                                                  bf16* __restrict__ m, long ldm, int f, int swiglu) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  const long row = blockIdx.y;
  const int c0 = (blockIdx.x * ACT_CH * 128 + threadIdx.x) * 8;
  uint4 gv[ACT_CH], uv[ACT_CH];
#pragma unroll
  for (int k = 0; k < ACT_CH; ++k) {
    const int c = c0 + k * 128 * 8;
    gv[k] = uv[k] = make_uint4(0, 0, 0, 0);
    if (c < f) {
      gv[k] = __ldg(reinterpret_cast<const uint4*>(gu + row * ld_gu + c));
      if (swiglu) uv[k] = __ldg(reinterpret_cast<const uint4*>(gu + row * ld_gu + f + c));
    }
  }
#pragma unroll
  for (int k = 0; k < ACT_CH; ++k) {
    const int c = c0 + k * 128 * 8;
    if (c >= ldm) break;
    uint4 ov = make_uint4(0, 0, 0, 0);
    if (c < f) {
      const bf16* g = reinterpret_cast<const bf16*>(&gv[k]);
      const bf16* u = reinterpret_cast<const bf16*>(&uv[k]);
      uint32_t* o = reinterpret_cast<uint32_t*>(&ov);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float g0 = __bfloat162float(g[2 * i]), g1 = __bfloat162float(g[2 * i + 1]);
        o[i] = swiglu ? pack_bf16(silu_f(g0) * __bfloat162float(u[2 * i]),
                                  silu_f(g1) * __bfloat162float(u[2 * i + 1]))
                      : pack_bf16(fmaxf(g0, 0.f), fmaxf(g1, 0.f));
      }
    }
    *reinterpret_cast<uint4*>(m + row * ldm + c) = ov;
  }
}
void act_fwd(const bf16* gu, long ld_gu, bf16* m, long ldm, int rows, int f, int swiglu,
             cudaStream_t st) {
  if (rows <= 0) return;
  dim3 grid((unsigned)((ldm / 8 + 128 * ACT_CH - 1) / (128 * ACT_CH)), rows);
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(act_kernel, dim3(grid), dim3(128), 0, st, gu, ld_gu, m, ldm, f, swiglu);
}

__global__ void lora_pack_kernel(const float* __restrict__ lu, int r, bf16* __restrict__ m,
                                 long ldm, int f, int rows) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * r) return;
  const int row = t / r, j = t % r;
  m[(long)row * ldm + f + j] = __float2bfloat16(lu[(long)row * r + j]);
}
void lora_pack(const float* lu, int r, bf16* m, long ldm, int f, int rows, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  if (rows > 0) launch_pdl(lora_pack_kernel, dim3((rows * r + 255) / 256), dim3(256), 0, st, lu, r, m, ldm, f, rows);
}

// ---------------------------------------------------------------- sampling / CE
// greedy sampling: stage 1 = (row, chunk) blocks with float4 loads, each the max of an
// order-preserving key (value bits << 32 | ~index: ties -> smallest index); stage 2 = one
// warp per row over the chunk keys.  Deterministic, no atomics.
constexpr int AMAX_CHUNKS = 16;
CS_DEV unsigned long long amax_key(float v, int i) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)o << 32) | (uint32_t)(0xFFFFFFFFu - (uint32_t)i);
}
__global__ void __launch_bounds__(256) argmax_part_kernel(const float* __restrict__ logits, long ld,
                                                          int V, unsigned long long* __restrict__ part) {
  __shared__ unsigned long long red[8];
  const float* row = logits + (long)blockIdx.x * ld;
  const int per = ((V + AMAX_CHUNKS - 1) / AMAX_CHUNKS + 3) & ~3;
  const int c0 = blockIdx.y * per, c1 = min(V, c0 + per);
  unsigned long long best = 0;
  const bool vec = (ld % 4) == 0;
  for (int c = c0 + threadIdx.x * 4; c < c1; c += blockDim.x * 4) {
    if (vec && c + 3 < c1) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(row + c));
      best = max(best, amax_key(v.x, c));
      best = max(best, amax_key(v.y, c + 1));
      best = max(best, amax_key(v.z, c + 2));
      best = max(best, amax_key(v.w, c + 3));
    } else {
      for (int k = c; k < min(c + 4, c1); ++k) best = max(best, amax_key(row[k], k));
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) best = max(best, red[i]);
    part[(long)blockIdx.x * AMAX_CHUNKS + blockIdx.y] = best;
  }
}
__global__ void argmax_final_kernel(const unsigned long long* __restrict__ part, int rows, int* out) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= rows) return;
  unsigned long long k = lane < AMAX_CHUNKS ? part[(long)row * AMAX_CHUNKS + lane] : 0ull;
  for (int o = 16; o > 0; o >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, o));
  if (lane == 0) out[row] = (int)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
}
void argmax_rows(const float* logits, long ld, int rows, int V, int* out,
                 unsigned long long* scratch, cudaStream_t st) {
  if (rows <= 0) return;
  cs::g_launches.fetch_add(2, std::memory_order_relaxed);
  argmax_part_kernel<<<dim3(rows, AMAX_CHUNKS), 256, 0, st>>>(logits, ld, V, scratch);
  argmax_final_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(scratch, rows, out);
}

__global__ void __launch_bounds__(512) ce_kernel(const float* __restrict__ logits, long ld,
                                                 const int* __restrict__ tg, int V, float inv_norm,
                                                 float* __restrict__ loss, bf16* __restrict__ dlog,
                                                 long ldd) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  __shared__ float red_m[16], red_s[16];
  const int row = blockIdx.x;
  const float* x = logits + (long)row * ld;
  bf16* dx = dlog + (long)row * ldd;
  const int t = tg[row];
  const int V4 = V & ~3;
  if (t < 0) {
    for (int c = threadIdx.x * 4; c < V4; c += blockDim.x * 4)
      *reinterpret_cast<uint2*>(dx + c) = make_uint2(0u, 0u);
    for (int c = V4 + threadIdx.x; c < V; c += blockDim.x) dx[c] = __float2bfloat16(0.f);
    if (threadIdx.x == 0) loss[row] = 0.f;
    return;
  }
  // pass 1: per-thread online (max, sum exp) over float4 slices, then a block merge
  float m = -INFINITY, se = 0.f;
  auto add = [&](float v) {
    if (v > m) {
      se = se * __expf(m - v) + 1.f;
      m = v;
    } else {
      se += __expf(v - m);
    }
  };
  for (int c = threadIdx.x * 4; c < V4; c += blockDim.x * 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(x + c));
    const float mv = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
    if (mv > m) {
      se *= __expf(m - mv);
      m = mv;
    }
    se += __expf(v.x - m) + __expf(v.y - m) + __expf(v.z - m) + __expf(v.w - m);
  }
  for (int c = V4 + threadIdx.x; c < V; c += blockDim.x) add(x[c]);
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, se, o);
    const float nm = fmaxf(m, om);
    se = (m == -INFINITY ? 0.f : se * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    m = nm;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red_m[w] = m;
    red_s[w] = se;
  }
  __syncthreads();
  float M = -INFINITY;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) M = fmaxf(M, red_m[i]);
  float S = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
    S += red_m[i] == -INFINITY ? 0.f : red_s[i] * __expf(red_m[i] - M);
  // pass 2: dlogits = (softmax - onehot) / (L-1) in bf16
  const float inv = 1.f / S;
  for (int c = threadIdx.x * 4; c < V4; c += blockDim.x * 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(x + c));
    float g0 = __expf(v.x - M) * inv, g1 = __expf(v.y - M) * inv;
    float g2 = __expf(v.z - M) * inv, g3 = __expf(v.w - M) * inv;
    if (t >= c && t < c + 4) {
      if (t == c) g0 -= 1.f;
      if (t == c + 1) g1 -= 1.f;
      if (t == c + 2) g2 -= 1.f;
      if (t == c + 3) g3 -= 1.f;
    }
    *reinterpret_cast<uint2*>(dx + c) =
        make_uint2(pack_bf16(g0 * inv_norm, g1 * inv_norm), pack_bf16(g2 * inv_norm, g3 * inv_norm));
  }
  for (int c = V4 + threadIdx.x; c < V; c += blockDim.x) {
    float g = __expf(x[c] - M) * inv;
    if (c == t) g -= 1.f;
    dx[c] = __float2bfloat16(g * inv_norm);
  }
  if (threadIdx.x == 0) loss[row] = (M + __logf(S)) - x[t];
}
void ce_fwd_bwd(const float* logits, long ld, const int* targets, int rows, int V,
                float inv_norm, float* loss, bf16* dlogits, long ldd, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  if (rows > 0) launch_pdl(ce_kernel, dim3(rows), dim3(512), 0, st, logits, ld, targets, V, inv_norm, loss, dlogits, ldd);
}

// ---------------------------------------------------------------- backward helpers
// RMSNorm backward + residual add, one 256-thread block per row; the row's dY, x (and the
// residual) are read once into registers (float4, <= 8 per thread: h <= 8192) and reused for
// the dot product and the output.
// (float4 registers sized for the row: h <= 4096 uses the V = 4 instance, 4 blocks per SM
// resident instead of 2 -- a 2048-row window ran at 50% of HBM with 23% of warps active)
constexpr int RMSB_V = 8;
template <int V>
__global__ void __launch_bounds__(256, V == 4 ? 4 : 2) rms_bwd_kernel(const float* __restrict__ resid, long ldr,
                               const float* __restrict__ x, long ldx, const float* __restrict__ g,
                               const float* __restrict__ rstd, const float* __restrict__ dh,
                               long ldh, float* __restrict__ out, long ldo, bf16* __restrict__ ob,
                               long ldob, int h, int use_norm) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  __shared__ float red[32];
  const long row = blockIdx.x;
  const float* dr = dh + row * ldh;
  const float* rr = resid ? resid + row * ldr : nullptr;
  float* o = out + row * ldo;
  float4 vd[V], vx[V], vr[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int c = (threadIdx.x + k * 256) * 4;
    vd[k] = vx[k] = vr[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < h) {
      vd[k] = __ldg(reinterpret_cast<const float4*>(dr + c));
      if (use_norm) vx[k] = __ldg(reinterpret_cast<const float4*>(x + row * ldx + c));
      if (rr) vr[k] = __ldg(reinterpret_cast<const float4*>(rr + c));
    }
  }
  float rs = 1.f, dot = 0.f;
  if (use_norm) {
    rs = rstd[row];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int c = (threadIdx.x + k * 256) * 4;
      if (c < h) {
        const float4 gg = __ldg(reinterpret_cast<const float4*>(g + c));
        dot += vd[k].x * gg.x * vx[k].x + vd[k].y * gg.y * vx[k].y + vd[k].z * gg.z * vx[k].z +
               vd[k].w * gg.w * vx[k].w;
      }
    }
    dot = block_sum(dot * rs, red) / (float)h;
  }
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int c = (threadIdx.x + k * 256) * 4;
    if (c >= h) continue;
    float4 v;
    if (use_norm) {
      const float4 gg = __ldg(reinterpret_cast<const float4*>(g + c));
      v.x = vr[k].x + rs * (vd[k].x * gg.x - vx[k].x * rs * dot);
      v.y = vr[k].y + rs * (vd[k].y * gg.y - vx[k].y * rs * dot);
      v.z = vr[k].z + rs * (vd[k].z * gg.z - vx[k].z * rs * dot);
      v.w = vr[k].w + rs * (vd[k].w * gg.w - vx[k].w * rs * dot);
    } else {
      v = make_float4(vr[k].x + vd[k].x, vr[k].y + vd[k].y, vr[k].z + vd[k].z, vr[k].w + vd[k].w);
    }
    *reinterpret_cast<float4*>(o + c) = v;
    if (ob) *reinterpret_cast<uint2*>(ob + row * ldob + c) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}
void rms_bwd_add(const float* resid, long ldr, const float* x, long ldx, const float* g,
                 const float* rstd, const float* dh, long ldh, float* out, long ldo,
                 bf16* out_b, long ldob, int rows, int h, int use_norm, cudaStream_t st) {
  if (rows <= 0) return;
  if (h > RMSB_V * 1024 || (h % 4) != 0) return;  // engine_create bounds h (multiple of 64)
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(h <= 4096 ? rms_bwd_kernel<4> : rms_bwd_kernel<RMSB_V>, dim3(rows), dim3(256), 0, st, resid, ldr, x, ldx, g,
             rstd, dh, ldh, out, ldo, out_b,
                                       ldob, h, use_norm);
}

// MLP backward fused with the LoRA-A gradient:
//   swiglu: saved / dgu in the interleaved gate||up layout (kernels.h EPI_SWIGLU: column j's
//           gate at (j/64)*128 + j%64, its up 64 further); dgu_gate = dm*u*dsilu(g),
//           dgu_up = dm*silu(g); m = silu(g)*u
//   relu  : m=saved;  dgu = dm * (m > 0)            (tiny_model.hpp:285-286)
//   dA[col, :] += sum_rows m[row, col] * dlu[row, :] (tiny_model.hpp:282)
// HBM-bound (10 B per (row, col): dm bf16 in, g / u bf16 in, dgu bf16 out).  Thread = 4
// adjacent columns (16-B / 8-B accesses), block = 128 threads x 512 columns x 256 rows; rows
// are processed in pairs with both rows' loads issued before either is used (memory-level
// parallelism), sigmoid on the SFU (ex2 + rcp), the dA partial sums on FFMA2 (column pairs),
// float4 atomics at the end (ncu: 467 -> 313 us per 8192-row window at the 8B shape; the
// 2-column variant at full occupancy measured 360 us).
constexpr int MLP_ROWS = 256;
constexpr int MLP_THREADS = 128;
__global__ void __launch_bounds__(MLP_THREADS) mlp_bwd_kernel(const bf16* __restrict__ dm, long ld_dm,
                                                              const bf16* __restrict__ saved, long ld_s,
                                                              const float* __restrict__ dlu, int r,
                                                              bf16* __restrict__ dgu, long ld_dgu,
                                                              float* __restrict__ dA, int rows, int f,
                                                              int swiglu) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  __shared__ __align__(16) float sl[MLP_ROWS * 16];
  const int col = 4 * (blockIdx.x * MLP_THREADS + threadIdx.x);
  const int rpb = (rows + gridDim.y - 1) / gridDim.y;  // rows per block (<= MLP_ROWS)
  const int r0 = blockIdx.y * rpb;
  const int nr = max(0, min(rpb, rows - r0));
  for (int i = threadIdx.x; i < nr * 16; i += MLP_THREADS) {
    const int rr = i >> 4, j = i & 15;
    sl[i] = j < r ? dlu[(long)(r0 + rr) * r + j] : 0.f;
  }
  __syncthreads();
  if (col >= f) return;
  float2 acc01[16], acc23[16];  // columns (col, col+1) and (col+2, col+3) per LoRA rank j
#pragma unroll
  for (int j = 0; j < 16; ++j) acc01[j] = acc23[j] = make_float2(0.f, 0.f);
  auto body = [&](int i, const float4& d, const uint2& gv, const uint2& uv) {
    float m[4], o0[4], o1[4];
    const float dd[4] = {d.x, d.y, d.z, d.w};
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const float g[4] = {__low2float(g2[0]), __high2float(g2[0]), __low2float(g2[1]), __high2float(g2[1])};
    if (swiglu) {
      const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
      const float u[4] = {__low2float(u2[0]), __high2float(u2[0]), __low2float(u2[1]), __high2float(u2[1])};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float sgm = sigmoid_f(g[q]);
        const float sl = g[q] * sgm;                                   // silu(g)
        m[q] = sl * u[q];
        o0[q] = dd[q] * u[q] * (sgm * (1.f + g[q] * (1.f - sgm)));   // dsilu(g)
        o1[q] = dd[q] * sl;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        m[q] = fmaxf(g[q], 0.f);
        o0[q] = m[q] > 0.f ? dd[q] : 0.f;
        o1[q] = 0.f;
      }
    }
    const long row = r0 + i;
    const int gc = swiglu ? (col >> 6) * 128 + (col & 63) : col;
    *reinterpret_cast<uint2*>(dgu + row * ld_dgu + gc) = make_uint2(pack_bf16(o0[0], o0[1]), pack_bf16(o0[2], o0[3]));
    if (swiglu)
      *reinterpret_cast<uint2*>(dgu + row * ld_dgu + gc + 64) =
          make_uint2(pack_bf16(o1[0], o1[1]), pack_bf16(o1[2], o1[3]));
    const float2 m01 = make_float2(m[0], m[1]), m23 = make_float2(m[2], m[3]);
    const float4* l4 = reinterpret_cast<const float4*>(sl + i * 16);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 l = l4[q];
      acc01[4 * q] = ffma2(m01, make_float2(l.x, l.x), acc01[4 * q]);
      acc23[4 * q] = ffma2(m23, make_float2(l.x, l.x), acc23[4 * q]);
      acc01[4 * q + 1] = ffma2(m01, make_float2(l.y, l.y), acc01[4 * q + 1]);
      acc23[4 * q + 1] = ffma2(m23, make_float2(l.y, l.y), acc23[4 * q + 1]);
      acc01[4 * q + 2] = ffma2(m01, make_float2(l.z, l.z), acc01[4 * q + 2]);
      acc23[4 * q + 2] = ffma2(m23, make_float2(l.z, l.z), acc23[4 * q + 2]);
      acc01[4 * q + 3] = ffma2(m01, make_float2(l.w, l.w), acc01[4 * q + 3]);
      acc23[4 * q + 3] = ffma2(m23, make_float2(l.w, l.w), acc23[4 * q + 3]);
    }
  };
  auto ld = [&](int i, float4& d, uint2& gv, uint2& uv) {
    const long row = r0 + i;
    const uint2 dv = __ldg(reinterpret_cast<const uint2*>(dm + row * ld_dm + col));
    const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
    d = make_float4(__low2float(d2[0]), __high2float(d2[0]), __low2float(d2[1]), __high2float(d2[1]));
    const int gc = swiglu ? (col >> 6) * 128 + (col & 63) : col;
    gv = __ldg(reinterpret_cast<const uint2*>(saved + row * ld_s + gc));
    uv = swiglu ? __ldg(reinterpret_cast<const uint2*>(saved + row * ld_s + gc + 64)) : make_uint2(0u, 0u);
  };
  int i = 0;
  for (; i + 3 < nr; i += 4) {  // four rows' loads in flight before any is used
    float4 d0, d1, d2, d3;
    uint2 g0, g1, g2, g3, u0, u1, u2, u3;
    ld(i, d0, g0, u0);
    ld(i + 1, d1, g1, u1);
    ld(i + 2, d2, g2, u2);
    ld(i + 3, d3, g3, u3);
    body(i, d0, g0, u0);
    body(i + 1, d1, g1, u1);
    body(i + 2, d2, g2, u2);
    body(i + 3, d3, g3, u3);
  }
  for (; i < nr; ++i) {
    float4 d0;
    uint2 g0, u0;
    ld(i, d0, g0, u0);
    body(i, d0, g0, u0);
  }
  // dA rows col..col+3, ranks j: float4 atomics over j (dA is [f, r] row-major, r <= 16)
  auto flush = [&](int q, float* dst) {
    auto val = [&](int j) { return q == 0 ? acc01[j].x : q == 1 ? acc01[j].y : q == 2 ? acc23[j].x : acc23[j].y; };
    if (r == 16) {
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        atomicAdd(reinterpret_cast<float4*>(dst + j), make_float4(val(j), val(j + 1), val(j + 2), val(j + 3)));
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < r) atomicAdd(dst + j, val(j));
    }
  };
#pragma unroll
  for (int q = 0; q < 4; ++q) flush(q, dA + (long)(col + q) * r);
}
void mlp_bwd(const bf16* dm, long ld_dm, const bf16* saved, long ld_s, const float* dlu, int r,
             bf16* dgu, long ld_dgu, float* dA, int rows, int f, int swiglu, cudaStream_t st) {
  if (rows <= 0) return;
  // enough blocks to keep ~6 per SM streaming (a 2048-row window on 256-row blocks ran 224
  // blocks: 9% warps active, 30% of HBM; ncu profiles/r2_elem_bwd_ncu.txt), <= MLP_ROWS rows each
  const int gx = (f / 4 + MLP_THREADS - 1) / MLP_THREADS;
  const int gy = std::max((rows + MLP_ROWS - 1) / MLP_ROWS,
                          std::min((rows + 31) / 32, (6 * 148 + gx - 1) / gx));
  dim3 grid(gx, gy);
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(mlp_bwd_kernel, dim3(grid), dim3(MLP_THREADS), 0, st, dm, ld_dm, saved, ld_s, dlu, r, dgu, ld_dgu, dA, rows, f,
                                               swiglu);
}

// dB[j, c] += sum_rows lu[row, j] * dY[row, c]  (tiny_model.hpp:280); 4 columns per thread
// (one float4 of dY per row), 128 threads x 512 columns x 64 rows per block (8 x s/64 blocks:
// enough CTAs to fill the SMs at every window size), FFMA2 on column pairs, float4 atomics.
// The same pass writes dycat[:, :h] = bf16(dY), the A operand of the dlu and dm GEMMs (its
// LoRA columns are filled by lora_pack, its pad columns stay zero from engine creation):
// one read of the fp32 dY instead of two
constexpr int LDB_ROWS = 64;
__global__ void __launch_bounds__(128) lora_db_kernel(const float* __restrict__ dY, long ldy,
                                                      const float* __restrict__ lu, int r,
                                                      int rows, int h, float* __restrict__ dB,
                                                      bf16* __restrict__ dycat, long ldc) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  __shared__ __align__(16) float sl[LDB_ROWS * 16];
  const int col = 4 * (blockIdx.x * 128 + threadIdx.x);
  const int r0 = blockIdx.y * LDB_ROWS;
  const int nr = min(LDB_ROWS, rows - r0);
  for (int i = threadIdx.x; i < nr * 16; i += 128) {
    const int rr = i >> 4, j = i & 15;
    sl[i] = j < r ? lu[(long)(r0 + rr) * r + j] : 0.f;
  }
  __syncthreads();
  if (col >= h) return;
  float2 a01[16], a23[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a01[j] = a23[j] = make_float2(0.f, 0.f);
  auto row = [&](int i, const float4& v) {
    *reinterpret_cast<uint2*>(dycat + (long)(r0 + i) * ldc + col) =
        make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
    const float2 v01 = make_float2(v.x, v.y), v23 = make_float2(v.z, v.w);
    const float4* l4 = reinterpret_cast<const float4*>(sl + i * 16);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 l = l4[q];
      const float lj[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a01[4 * q + t] = ffma2(v01, make_float2(lj[t], lj[t]), a01[4 * q + t]);
        a23[4 * q + t] = ffma2(v23, make_float2(lj[t], lj[t]), a23[4 * q + t]);
      }
    }
  };
  const float* yp = dY + (long)r0 * ldy + col;
  int i = 0;
  for (; i + 3 < nr; i += 4) {  // four rows' loads in flight before any is used
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(yp + (long)i * ldy));
    const float4 v1 = __ldg(reinterpret_cast<const float4*>(yp + (long)(i + 1) * ldy));
    const float4 v2 = __ldg(reinterpret_cast<const float4*>(yp + (long)(i + 2) * ldy));
    const float4 v3 = __ldg(reinterpret_cast<const float4*>(yp + (long)(i + 3) * ldy));
    row(i, v0);
    row(i + 1, v1);
    row(i + 2, v2);
    row(i + 3, v3);
  }
  for (; i < nr; ++i) row(i, __ldg(reinterpret_cast<const float4*>(yp + (long)i * ldy)));
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < r)
      atomicAdd(reinterpret_cast<float4*>(dB + (long)j * h + col),
                make_float4(a01[j].x, a01[j].y, a23[j].x, a23[j].y));
}
void lora_db(const float* dY, long ldy, const float* lu, int r, int rows, int h, float* dB,
             bf16* dycat, long ldc, cudaStream_t st) {
  if (rows <= 0) return;
  dim3 grid((h / 4 + 127) / 128, (rows + LDB_ROWS - 1) / LDB_ROWS);
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(lora_db_kernel, dim3(grid), dim3(128), 0, st, dY, ldy, lu, r, rows, h, dB, dycat, ldc);
}

// inverse (transposed) rotate-half RoPE + pack [dq | dk | dv] as bf16
__global__ void rope_bwd_pack_kernel(const float* __restrict__ dq, long ldq,
                                     const float* __restrict__ dk, const float* __restrict__ dv,
                                     long ld_acc, int a, int n_heads, int n_kv, int d,
                                     int use_rope, const float2* __restrict__ tab,
                                     bf16* __restrict__ out, long ldo) {
  griddep_launch();  // PDL: a dependent GEMM may start its weight prefetch now
  griddep_wait();    // launched with PDL: the producer's writes are visible from here on
  const int i = blockIdx.x;  // window-local row
  const int pos = a + i;
  const int half = d / 2;
  const int q_dim = n_heads * d, kv_dim = n_kv * d;
  bf16* o = out + (long)i * ldo;
  // 4 consecutive rotation pairs per thread (d / 2 is a multiple of 4): 16-byte loads of both
  // halves and of the table, 8-byte bf16 stores
  const int nqp = n_heads * half / 4, nkp = n_kv * half / 4;
  for (int t = threadIdx.x; t < nqp + nkp; t += blockDim.x) {
    const bool isq = t < nqp;
    const int tt = (isq ? t : t - nqp) * 4;
    const int hd = tt / half, j = tt % half;
    const float* src = isq ? dq + (long)i * ldq + hd * d : dk + (long)pos * ld_acc + hd * d;
    const float4 a1 = *reinterpret_cast<const float4*>(src + j);
    const float4 a2 = *reinterpret_cast<const float4*>(src + j + half);
    float y1[4] = {a1.x, a1.y, a1.z, a1.w}, y2[4] = {a2.x, a2.y, a2.z, a2.w};
    if (use_rope) {
      const float4* tp = reinterpret_cast<const float4*>(tab + (long)pos * half + j);
      const float4 c01 = tp[0], c23 = tp[1];
      const float cx[4] = {c01.x, c01.z, c23.x, c23.z}, cy[4] = {c01.y, c01.w, c23.y, c23.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float x1 = y1[q] * cx[q] + y2[q] * cy[q];
        const float x2 = y2[q] * cx[q] - y1[q] * cy[q];
        y1[q] = x1;
        y2[q] = x2;
      }
    }
    bf16* dst = o + (isq ? 0 : q_dim) + hd * d;
    *reinterpret_cast<uint2*>(dst + j) = make_uint2(pack_bf16(y1[0], y1[1]), pack_bf16(y1[2], y1[3]));
    *reinterpret_cast<uint2*>(dst + j + half) = make_uint2(pack_bf16(y2[0], y2[1]), pack_bf16(y2[2], y2[3]));
  }
  for (int c = threadIdx.x * 4; c < kv_dim; c += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(dv + (long)pos * ld_acc + c);
    *reinterpret_cast<uint2*>(o + q_dim + kv_dim + c) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}
void rope_bwd_pack(const float* dq, long ldq, const float* dk, const float* dv, long ld_acc,
                   int a, int rows, int n_heads, int n_kv_heads, int head_dim, int use_rope,
                   float theta, bf16* out, long ldo, cudaStream_t st) {
  (void)theta;
  if (rows <= 0) return;
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  launch_pdl(rope_bwd_pack_kernel, dim3(rows), dim3(128), 0, st, dq, ldq, dk, dv, ld_acc, a, n_heads, n_kv_heads,
             head_dim, use_rope, s_rope_tab, out, ldo);
}

// ---------------------------------------------------------------- Adam (fp32 master)
__global__ void adam_kernel(AdamParams p, int update) {
  const long nA = (long)p.n_layers * p.f * p.r;
  const long nB = (long)p.n_layers * p.r * p.h;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < nA + nB;
       t += (long)gridDim.x * blockDim.x) {
    const bool isA = t < nA;
    const long i = isA ? t : t - nA;
    float* w = isA ? p.A + i : p.B + i;
    if (update) {
      const float g = isA ? p.gA[i] : p.gB[i];
      float* m = isA ? p.mA + i : p.mB + i;
      float* v = isA ? p.vA + i : p.vB + i;
      const float mm = p.b1 * *m + (1.f - p.b1) * g;
      const float vv = p.b2 * *v + (1.f - p.b2) * g * g;
      *m = mm;
      *v = vv;
      const float mh = mm / p.bc1, vh = vv / p.bc2;
      *w = *w - p.lr * mh / (sqrtf(vh) + p.eps);
    }
    const bf16 wb = __float2bfloat16(*w);
    if (isA) {  // A[l][row][j]
      const long l = i / ((long)p.f * p.r);
      const long rem = i % ((long)p.f * p.r);
      const int row = (int)(rem / p.r), j = (int)(rem % p.r);
      p.A_t[(l * 16 + j) * p.f + row] = wb;  // [n_layers][16][f]
      p.down_cat[(l * p.down_rows + p.h + j) * (p.f + 64) + row] = wb;
    } else {    // B[l][j][c]
      const long l = i / ((long)p.r * p.h);
      const long rem = i % ((long)p.r * p.h);
      const int j = (int)(rem / p.h), c = (int)(rem % p.h);
      p.down_cat[(l * p.down_rows + c) * (p.f + 64) + p.f + j] = wb;
      p.B_t[(l * 16 + j) * p.h + c] = wb;  // [n_layers][16][h]
    }
  }
}
void adam_step(const AdamParams& p, int update, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  adam_kernel<<<4 * 148, 256, 0, st>>>(p, update);
}

// ---------------------------------------------------------------- weight prep
// transpose: dst row = c, mapped through 64-row blocks when blk_stride > 0 (the interleaved
// gate||up layout: row (c / 64) * blk_stride + blk_off + c % 64)
__global__ void cast_kernel(const float* __restrict__ src, int rows, int cols, bf16* dst,
                            long ldd, int transpose, int blk_stride, int blk_off) {
  __shared__ float tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int k = 0; k < 32; k += 8) {
    const int r = by + ty + k, c = bx + tx;
    if (r < rows && c < cols) {
      if (!transpose) dst[(long)r * ldd + c] = __float2bfloat16(src[(long)r * cols + c]);
      else tile[ty + k][tx] = src[(long)r * cols + c];
    }
  }
  if (!transpose) return;
  __syncthreads();
  for (int k = 0; k < 32; k += 8) {
    const int c = bx + ty + k, r = by + tx;  // dst row = c, dst col = r
    const long dr = blk_stride > 0 ? (long)(c >> 6) * blk_stride + blk_off + (c & 63) : c;
    if (r < rows && c < cols) dst[dr * ldd + r] = __float2bfloat16(tile[tx][ty + k]);
  }
}
void cast_f32_bf16(const float* src, int rows, int cols, bf16* dst, long ldd, int transpose,
                   cudaStream_t st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  cast_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, dst, ldd, transpose, 0, 0);
}
void cast_f32_bf16_interleaved(const float* src, int rows, int cols, bf16* dst, long ldd, int blk_stride,
                               int blk_off, cudaStream_t st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  cast_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, dst, ldd, 1, blk_stride, blk_off);
}

CS_DEV uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
CS_DEV float hash_normal(uint64_t seed, long i) {
  const uint64_t a = splitmix(seed ^ splitmix((uint64_t)i * 2 + 1));
  const float u1 = ((a >> 40) + 1) * (1.0f / 16777217.0f);
  const float u2 = (a & 0xFFFFFF) * (1.0f / 16777216.0f);
  return sqrtf(-2.f * __logf(u1)) * __cosf(6.2831853f * u2);
}
__global__ void init_bf16_kernel(bf16* dst, long n, float scale, uint64_t seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16(hash_normal(seed, i) * scale);
}
__global__ void init_f32_kernel(float* dst, long n, float scale, uint64_t seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = hash_normal(seed, i) * scale;
}
__global__ void fill_kernel(float* dst, long n, float v) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = v;
}
void init_normal_bf16(bf16* dst, long n, float scale, uint64_t seed, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  init_bf16_kernel<<<8 * 148, 256, 0, st>>>(dst, n, scale, seed);
}
void init_normal_f32(float* dst, long n, float scale, uint64_t seed, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  init_f32_kernel<<<8 * 148, 256, 0, st>>>(dst, n, scale, seed);
}
void fill_f32(float* dst, long n, float v, cudaStream_t st) {
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  fill_kernel<<<4 * 148, 256, 0, st>>>(dst, n, v);
}

}  // namespace cs
