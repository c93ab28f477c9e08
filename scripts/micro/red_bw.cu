// red_bw.cu -- micro-benchmark: L2 fp32 reduce-add throughput of cp.reduce.async.bulk (smem ->
// global .add.f32) in the attention-backward dQ pattern: every CTA (one per SM) adds a 32 KB
// tile per step as `chunks` bulk ops, CTA c at step t targeting tile (c * stride + t) of a
// `region_mb` fp32 buffer (CTAs sweep the buffer at offset positions, as the key-tile CTAs of the
// backward sweep the query tiles).  Reports GB/s of reduced bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 red_bw.cu -o red_bw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2402_18789_b200/csrc/common.cuh"
using namespace cs;

__global__ void __launch_bounds__(128, 1) red(float* buf, long n_tiles, int steps, int chunks, int stride,
                                              int depth) {
  extern __shared__ __align__(1024) uint8_t smem[];
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int cb = 32768 / chunks;
    for (int t = 0; t < steps; ++t) {
      const long tile = ((long)blockIdx.x * stride + t) % n_tiles;
      char* dst = reinterpret_cast<char*>(buf) + tile * 32768;
      for (int c = 0; c < chunks; ++c)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                         dst + c * cb),
                     "r"(smem_u32(smem + c * cb)), "r"(cb)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (depth == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
}

// per-thread warp-coalesced red.global.add.f32: a 32 KB tile = 64 rows x 128 floats, warp w of
// `nw` covers columns [32 (w % 4), +32) of rows w / 4, w / 4 + nw / 4, ... (128 B per warp instruction)
__global__ void red_warp(float* buf, long n_tiles, int steps, int stride, int v2) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int t = 0; t < steps; ++t) {
    const long tile = ((long)blockIdx.x * stride + t) % n_tiles;
    float* base = buf + tile * 8192;
    if (!v2) {
      for (int r = w / 4; r < 64; r += nw / 4)
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(base + r * 128 + (w % 4) * 32 + lane), "f"(1.0f) : "memory");
    } else {
      for (int r = w / 4; r < 64; r += nw / 4)
        if (lane < 16)
          asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(base + r * 128 + (w % 4) * 32 + 2 * lane), "f"(1.0f), "f"(1.0f) : "memory");
    }
  }
}

int main() {
  {
    const long region = 128l << 20;
    float* b2;
    cudaMalloc(&b2, region);
    cudaMemset(b2, 0, region);
    cudaEvent_t a0, a1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    for (int nw : {4, 8, 16})
      for (int v2 : {0, 1}) {
        const int steps = 500;
        red_warp<<<148, nw * 32>>>(b2, region / 32768, 20, 8, v2);
        cudaEventRecord(a0);
        red_warp<<<148, nw * 32>>>(b2, region / 32768, steps, 8, v2);
        cudaEventRecord(a1);
        if (cudaEventSynchronize(a1) != cudaSuccess) { printf("fail\n"); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, a0, a1);
        const double bytes = 148.0 * steps * 32768 / (v2 ? 2 : 1);
        printf("red.global.add%s warps %2d: %7.1f GB/s reduced (%.3f ms)\n", v2 ? ".v2 (half the lanes)" : ".f32", nw,
               bytes / ms / 1e6, ms);
      }
  }
  const long region = 128l << 20;
  float* buf;
  cudaMalloc(&buf, region);
  cudaMemset(buf, 0, region);
  cudaFuncSetAttribute(red, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct C { int region_mb, chunks, stride, depth, ctas; };
  const C cs_[] = {{128, 16, 8, 1, 148}, {128, 16, 8, 0, 148}, {128, 1, 8, 1, 148}, {128, 64, 8, 1, 148},
                   {32, 16, 8, 1, 148},  {128, 16, 8, 1, 296}, {128, 16, 0, 1, 148}, {1024, 16, 8, 1, 148}};
  for (const C& c : cs_) {
    float* b = buf;
    float* big = nullptr;
    if (c.region_mb > 128) { cudaMalloc(&big, (long)c.region_mb << 20); cudaMemset(big, 0, (long)c.region_mb << 20); b = big; }
    const long nt = ((long)c.region_mb << 20) / 32768;
    const int steps = 2000;
    red<<<c.ctas, 128, 32768>>>(b, nt, 50, c.chunks, c.stride, c.depth);
    cudaEventRecord(e0);
    red<<<c.ctas, 128, 32768>>>(b, nt, steps, c.chunks, c.stride, c.depth);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) { printf("fail\n"); return 1; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)c.ctas * steps * 32768;
    printf("region %5d MB  %2d ops/32KB  stride %d  depth %d  ctas %d: %7.1f GB/s reduced (%.3f ms)\n", c.region_mb,
           c.chunks, c.stride, c.depth, c.ctas, bytes / ms / 1e6, ms);
    if (big) cudaFree(big);
  }
  return 0;
}
