// TMA load throughput / latency microbenchmark (diagnostic, not product code):
// every CTA streams 32 KB tiles (2 boxes of [128 rows x 64 bf16], SWIZZLE_128B, row pitch
// `pitch` elements) from a buffer of `rows` rows through an S-stage mbarrier ring; reports
// B/clk/SM and the mean issue->arrival latency.  nvcc -arch=sm_100a -o tma_bw tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void __launch_bounds__(32, 1) tma_kernel(const __grid_constant__ CUtensorMap map, int rows, int iters,
                                                    unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(sm + S * 32768);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int ntile = rows / 128;
  unsigned long long t0 = clock64(), lat = 0;
  unsigned long long issue[8];
  auto load = [&](int i) {
    const int s = i % S;
    const int tile = (blockIdx.x * 7 + i) % ntile;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(32768) : "memory");
    for (int h = 0; h < 2; ++h)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(su32(sm + s * 32768 + h * 16384)), "l"((uint64_t)&map), "r"(su32(&bar[s])), "r"(h * 64), "r"(tile * 128) : "memory");
    issue[s] = clock64();
  };
  for (int i = 0; i < S; ++i) load(i);
  for (int i = 0; i < iters; ++i) {
    const int s = i % S;
    const uint32_t ph = (i / S) & 1;
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&bar[s])), "r"(ph) : "memory");
    lat += clock64() - issue[s];
    if (i + S < iters) load(i + S);
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * 2] = t1 - t0;
  out[blockIdx.x * 2 + 1] = lat / iters;
}

int main() {
  const long pitch = 1024;  // elements per row (kv_dim of the 8B model)
  const int rows = 8192 * 2;
  void* buf;
  cudaMalloc(&buf, (size_t)rows * pitch * 2);
  cudaMemset(buf, 1, (size_t)rows * pitch * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 2 * 8 * 4);
  std::vector<unsigned long long> h(148 * 2 * 4);
  for (int grid : {1, 148}) {
    auto run = [&](auto kern, int S) {
      const int smem = S * 32768 + 2048;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<grid, 32, smem>>>(map, rows, 200, out);  // warm L2
      kern<<<grid, 32, smem>>>(map, rows, 400, out);
      cudaDeviceSynchronize();
      cudaMemcpy(h.data(), out, grid * 2 * 8, cudaMemcpyDeviceToHost);
      double cyc = 0, lat = 0;
      for (int b = 0; b < grid; ++b) { cyc += h[b * 2]; lat += h[b * 2 + 1]; }
      cyc /= grid; lat /= grid;
      printf("grid %3d stages %d: %.1f B/clk/SM, mean latency %.0f clk (%s)\n", grid, S, 400.0 * 32768 / cyc, lat,
             cudaGetErrorString(cudaGetLastError()));
    };
    run(tma_kernel<1>, 1); run(tma_kernel<2>, 2); run(tma_kernel<4>, 4); run(tma_kernel<6>, 6);
  }
  return 0;
}
