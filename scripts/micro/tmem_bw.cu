// tmem_bw.cu -- micro-benchmark: TMEM read throughput (tcgen05.ld 32x32b) per SM with 4 / 8
// reader warps, tcgen05.mma (M=128, N=128, K=16, bf16, SS operands) rate alone, and both at once
// (readers on TMEM columns the MMAs do not touch).  One CTA per SM, all 148 SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2402_18789_b200/csrc tmem_bw.cu -lcuda
#include <cstdio>
#include <vector>
void sweep_main();

#include "../../paper_2402_18789_b200/csrc/common.cuh"

using namespace cs;

__global__ void __launch_bounds__(384, 1) bench(int n_readers, int ld_iters, int mma_iters, int ts,
                                                unsigned long long* out, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  unsigned long long t0 = clock64();
  uint32_t acc = 0;
  if (warp == 0) {
    if (lane == 0 && mma_iters > 0) {
      constexpr uint32_t id = idesc_bf16_f32(128, 128);
      const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
      for (int i = 0; i < mma_iters; ++i) {
        if (ts)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
              "r"(tmem + 128 + (i & 7) * 8), "l"(umma_desc_sw128(sb + (i & 3) * 32)), "r"(id), "r"(1));
        else
          mma_bf16(tmem, umma_desc_sw128(sa + (i & 3) * 32), umma_desc_sw128(sb + (i & 3) * 32), id, 1);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else if (warp >= 4 && warp < 4 + n_readers) {
    const int sub = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t base = tmem + ((uint32_t)(sub * 32) << 16) + 256 + ((warp - 4) >> 2) * 128;
    for (int it = 0; it < ld_iters; ++it) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(base + (it & 3) * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[j];
    }
  }
  unsigned long long t1 = clock64();
  if (acc == 0x12345678u) sink[0] = acc;
  __shared__ unsigned long long tmax[12];
  tmax[warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m0 = tmax[0], mr = 0;
    for (int w = 4; w < 4 + n_readers; ++w) mr = tmax[w] > mr ? tmax[w] : mr;
    out[blockIdx.x * 2] = m0;
    out[blockIdx.x * 2 + 1] = mr;
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


__global__ void __launch_bounds__(128, 1) mma_sweep(int n, int ts, int nacc, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 98304 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 2) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && lane == 0) {
    const uint32_t id = idesc_bf16_f32(128, n);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i % nacc) * n);
      if (ts)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                     "r"(tmem + 256 + (i & 7) * 8), "l"(umma_desc_sw128(sb + (i & 3) * 32)), "r"(id), "r"(1));
      else
        mma_bf16(d, umma_desc_sw128(sa + (i & 3) * 32), umma_desc_sw128(sb + (i & 3) * 32), id, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  sweep_main();
  unsigned long long* d_out;
  uint32_t* d_sink;
  cudaMalloc(&d_out, 148 * 2 * 8);
  cudaMalloc(&d_sink, 4);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  std::vector<unsigned long long> h(148 * 2);
  struct Cfg { const char* name; int nr, ldi, mmai, ts; };
  const Cfg cfgs[] = {
      {"ld 4 warps", 4, 4096, 0, 0},         {"ld 8 warps", 8, 4096, 0, 0},
      {"mma SS only", 0, 0, 8192, 0},         {"mma TS only", 0, 0, 8192, 1},
      {"mma SS + ld 4w", 4, 4096, 8192, 0},   {"mma SS + ld 8w", 8, 4096, 8192, 0},
      {"mma TS + ld 4w", 4, 4096, 8192, 1},   {"mma TS + ld 8w", 8, 4096, 8192, 1},
  };
  for (int rep = 0; rep < 2; ++rep)
    for (const Cfg& c : cfgs) {
      bench<<<148, 384, 66 * 1024 + 1024>>>(c.nr, c.ldi, c.mmai, c.ts, d_out, d_sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost);
      double m0 = 0, mr = 0;
      for (int b = 0; b < 148; ++b) { m0 += h[2 * b]; mr += h[2 * b + 1]; }
      m0 /= 148; mr /= 148;
      const double ld_bytes = (double)c.nr * c.ldi * 32 * 32 * 4;
      const double macs = (double)c.mmai * 128 * 128 * 16;
      if (rep == 1)
        printf("%-18s mma %9.0f clk (%6.0f MAC/clk)  ld %9.0f clk (%6.1f B/clk)\n", c.name, m0,
               m0 > 0 && c.mmai ? macs / m0 : 0.0, mr, mr > 0 && c.nr ? ld_bytes / mr : 0.0);
    }
  return 0;
}

void sweep_main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 148 * 8);
  cudaFuncSetAttribute(mma_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  std::vector<unsigned long long> h(148);
  for (int rep = 0; rep < 2; ++rep)
    for (int ts = 0; ts < 2; ++ts)
      for (int n : {32, 64, 128, 256})
        for (int nacc : {1, 2}) {
          if (ts && n * nacc > 256) continue;
          if (!ts && n * nacc > 512) continue;
          const int iters = 4096;
          mma_sweep<<<148, 128, 98304 + 1024>>>(n, ts, nacc, iters, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("sweep: %s\n", cudaGetErrorString(e)); exit(1); }
          cudaMemcpy(h.data(), d_out, 148 * 8, cudaMemcpyDeviceToHost);
          double m = 0; for (auto v : h) m += v; m /= 148;
          if (rep == 1) printf("M=128 N=%3d %s nacc=%d: %6.1f clk/mma  %6.0f MAC/clk\n", n, ts ? "TS" : "SS", nacc,
                               m / iters, 128.0 * n * 16 * iters / m);
        }
}
