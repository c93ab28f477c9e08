// mma_rate.cu -- tcgen05.mma issue / execution rate per SM for M=128, N in {64,128,256}, K=16 bf16,
// compile-time instruction descriptors, constant operand addresses, unrolled issue loop; NACC
// accumulators used round-robin.  One CTA per SM on all 148 SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_rate.cu -o mma_rate -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2402_18789_b200/csrc/common.cuh"
using namespace cs;

template <int N, int NACC, int TS>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 2) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && lane == 0) {
    constexpr uint32_t id = idesc_bf16_f32(128, N);
    const uint64_t da = umma_desc_sw128(smem_u32(smem)), db = umma_desc_sw128(smem_u32(smem + 32768));
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t d = tmem + (uint32_t)((j % NACC) * N);
        if (TS)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(tmem + 384), "l"(db), "r"(id), "r"(1));
        else
          mma_bf16(d, da, db, id, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, int NACC, int TS>
void run(const char* name) {
  static unsigned long long* d_out = nullptr;
  if (!d_out) cudaMalloc(&d_out, 148 * 8);
  cudaFuncSetAttribute(k<N, NACC, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  std::vector<unsigned long long> h(148);
  const int iters = 8192;
  for (int rep = 0; rep < 2; ++rep) {
    k<N, NACC, TS><<<148, 128, 65536 + 1024>>>(iters, d_out);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s failed\n", name); exit(1); }
  }
  cudaMemcpy(h.data(), d_out, 148 * 8, cudaMemcpyDeviceToHost);
  double m = 0; for (auto v : h) m += v; m /= 148;
  printf("%-22s %6.1f clk/mma  %6.0f MAC/clk/SM\n", name, m / iters, 128.0 * N * 16 * iters / m);
}


// the fused attention backward's per-tile MMA mix (attn_bwd2.cu), issued back to back by one
// thread with no waits: S^T, dP^T (8 + 8 SS, N=64, K-major), dV, dK (4 + 4 TS, N=128, B MN-major),
// dQ^T (8 SS, N=64, both MN-major) and the kernel's 4 commits per tile -- the tensor pipe's own
// floor for one (key block, query tile) pair
__global__ void __launch_bounds__(384, 1) tile_mix(int tiles, unsigned long long* out, int mode, int bg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[5];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 163840 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); stop = 0; }
  if (warp == 2) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // background traffic of the fused kernel's other warps (warps 4-11): bg 1 = tcgen05.ld of
  // 64 TMEM columns per pass (the elementwise warps' S / dP read-out), 2 = STS.128 + LDS.128
  // over a 32 KB smem region, 3 = both
  if (warp >= 4 && bg) {
    uint32_t acc = 0;
    uint4* sc = reinterpret_cast<uint4*>(smem + 163840) + (warp - 4) * 256 + lane;
    while (!stop) {
      if (bg & 1) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)((warp & 3) * 32) << 16), r);
        tmem_ld_32x32b_x32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + 32, r);
        tmem_ld_wait();
        acc += r[0] ^ r[31];
      }
      if (bg & 2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) sc[i * 32] = make_uint4(acc, i, 0, 0);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += sc[i * 32].y;
      }
    }
    if (acc == 0xdeadbeef) out[0] = acc;
  }
  if (warp == 0 && lane == 0) {
    constexpr uint32_t idS = idesc_bf16_f32_major(128, 64, 0, 0);
    constexpr uint32_t idG = idesc_bf16_f32_major(128, 128, 0, 1);
    constexpr uint32_t idQ = idesc_bf16_f32_major(128, 64, 1, 1);
    const uint32_t sK = smem_u32(smem), sV = sK + 32768, sQ = sK + 65536, sO = sK + 98304, sDS = sK + 131072;
    unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int t = 0; t < tiles; ++t) {
      if (mode != 2 && mode != 4) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ak = (kk >> 2) * 16384 + (kk & 3) * 32, bq = (kk >> 2) * 8192 + (kk & 3) * 32;
          mma_bf16(tmem + 0, umma_desc_sw128(sK + ak), umma_desc_sw128(sQ + bq), idS, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ak = (kk >> 2) * 16384 + (kk & 3) * 32, bq = (kk >> 2) * 8192 + (kk & 3) * 32;
          mma_bf16(tmem + 64, umma_desc_sw128(sV + ak), umma_desc_sw128(sO + bq), idS, kk > 0);
        }
        mma_commit(&bar[0]);
        if (mode == 3) { mbar_wait(&bar[0], ph); }
      }
      if (mode != 1) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem + 256),
                       "r"(tmem + 128 + kk * 8), "l"(umma_desc_sw128_mn(sO + kk * 2048, 8192, 1024)), "r"(idG), "r"(1));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem + 384),
                       "r"(tmem + 160 + kk * 8), "l"(umma_desc_sw128_mn(sQ + kk * 2048, 8192, 1024)), "r"(idG), "r"(1));
        mma_commit(&bar[1]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16(tmem + 192, umma_desc_sw128_mn(sK + kk * 2048, 16384, 1024),
                   umma_desc_sw128_mn(sDS + kk * 2048, 16384, 1024), idQ, kk > 0);
        mma_commit(&bar[2]);
        mma_commit(&bar[3]);
        if (mode >= 3) mbar_wait(&bar[3], ph);
      }
      ph ^= 1;
    }
    mma_commit(&bar[4]);
    mbar_wait(&bar[4], 0);
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

void run_mix(int mode, const char* name, int bg = 0) {
  static unsigned long long* d_out = nullptr;
  if (!d_out) cudaMalloc(&d_out, 148 * 8);
  cudaFuncSetAttribute(tile_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 163840 + 32768 + 1024);
  std::vector<unsigned long long> h(148);
  const int tiles = 2048;
  for (int rep = 0; rep < 2; ++rep) {
    tile_mix<<<148, 384, 163840 + 32768 + 1024>>>(tiles, d_out, mode, bg);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s failed\n", name); exit(1); }
  }
  cudaMemcpy(h.data(), d_out, 148 * 8, cudaMemcpyDeviceToHost);
  double m = 0; for (auto v : h) m += v; m /= 148;
  printf("%-34s %7.1f clk/tile\n", name, m / tiles);
}

int main() {
  run_mix(0, "bwd tile: S,dP + dV,dK,dQ^T");
  run_mix(1, "bwd tile: S,dP only");
  run_mix(2, "bwd tile: dV,dK,dQ^T only");
  run_mix(3, "serial: S,commit,wait; G,commit,wait");
  run_mix(4, "serial: G,commit,wait");
  run_mix(0, "bwd tile + 8 warps tcgen05.ld", 1);
  run_mix(0, "bwd tile + 8 warps STS/LDS", 2);
  run_mix(0, "bwd tile + 8 warps both", 3);
  run<64, 1, 0>("N=64  SS 1 acc");
  run<64, 2, 0>("N=64  SS 2 acc");
  run<64, 4, 0>("N=64  SS 4 acc");
  run<128, 1, 0>("N=128 SS 1 acc");
  run<128, 2, 0>("N=128 SS 2 acc");
  run<256, 1, 0>("N=256 SS 1 acc");
  run<64, 1, 1>("N=64  TS 1 acc");
  run<128, 1, 1>("N=128 TS 1 acc");
  run<256, 1, 1>("N=256 TS 1 acc");
  return 0;
}
