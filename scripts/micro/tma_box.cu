// tma_box.cu -- micro-benchmark: TMA load throughput per SM for the attention-backward Q / dO
// tile pattern (3D box {64 elems, 4 heads, 16 positions} over a [L][32 heads][128] bf16 tensor,
// SWIZZLE_128B) vs a 2D box of the same bytes ({64 elems, 64 rows} over [rows][128]); every CTA
// (one per SM) streams `tiles` tiles of 4 boxes (32 KB) through a `depth`-stage ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_box.cu -o tma_box -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>
#include "../../paper_2402_18789_b200/csrc/common.cuh"
using namespace cs;

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2,
                                            int three_d, int tiles,
                                            int n_pos_tiles, int depth, unsigned long long* out, int mma_mode) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[8];
  __shared__ uint64_t mbar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mbar_init(&full[i], 1);
    mbar_init(&mbar, 1);
    done = 0;
    fence_barrier_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x < 96) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // mma_mode 3: warps 2-3 keep storing to smem and issuing fence.proxy.async.shared::cta
  if (mma_mode == 3 && threadIdx.x >= 64) {
    uint32_t* w = reinterpret_cast<uint32_t*>(smem + 5 * 32768) + (threadIdx.x - 64) * 4;
    int it = 0;
    while (!done) {
      w[it & 3] = it;
      fence_proxy_async_smem();
      ++it;
    }
  }
  // concurrent tensor-core traffic: SS MMAs (M=128, N=64) over the last 2 stages of smem
  if (mma_mode && mma_mode < 3 && threadIdx.x == 32) {
    const uint32_t sa = smem_u32(smem + 4 * 32768), sb = smem_u32(smem + 5 * 32768);
    constexpr uint32_t id = idesc_bf16_f32(128, 64);
    int it = 0;
    while (!done) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        mma_bf16(slot, umma_desc_sw128(sa + (j & 3) * 32), umma_desc_sw128(sb + (j & 3) * 32), id, 1);
      if (mma_mode == 2 && (++it & 1)) __nanosleep(200);  // ~50% duty
    }
    mma_commit(&mbar);
    mbar_wait(&mbar, 0);
  }
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    auto issue = [&](int t) {
      const int st = t % depth;
      // mma_mode 4: every CTA reads the same tile sequence (L2 hot spot); 5: CTAs of 8 "heads"
      // start 8x tiles apart like the key-block CTAs of the backward
      const int pt = mma_mode == 4 ? t % n_pos_tiles
                   : mma_mode == 5 ? ((blockIdx.x / 8) * 8 + t) % n_pos_tiles
                                   : (blockIdx.x * 7 + t) % n_pos_tiles;  // position tile
      mbar_arrive_expect_tx(&full[st], 4 * 8192);
      for (int b = 0; b < 4; ++b) {
        uint8_t* dst = smem + st * 32768 + b * 8192;
        if (three_d)  // {64 elems, 4 heads, 16 positions}: (half b & 1, tensor b >> 1 in mode 6)
          tma_load_3d((mma_mode == 6 && (b >> 1)) ? &tm2 : &tm, &full[st], dst, (b & 1) * 64, (blockIdx.x % 8) * 4, pt * 16);
        else          // {64 elems, 64 rows}
          tma_load_2d(&tm, &full[st], dst, (b & 1) * 64, pt * 64 + (b >> 1) * 32768);
      }
    };
    for (int t = 0; t < depth && t < tiles; ++t) issue(t);
    for (int t = 0; t < tiles; ++t) {
      mbar_wait(&full[t % depth], (t / depth) & 1);
      if (t + depth < tiles) issue(t + depth);
    }
    out[blockIdx.x] = clock64() - t0;
    done = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x >= 64 && threadIdx.x < 96) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

int main() {
  const long L = 65536, H = 32;  // [L][32][128] bf16 = 512 MB (>> L2) or a prefix of it
  void* buf;
  cudaMalloc(&buf, L * H * 128 * 2);
  cudaMemset(buf, 0, L * H * 128 * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                           CUtensorMapFloatOOBfill)>(fn);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
  std::vector<unsigned long long> h(148);
  for (int mma_mode : {0, 6})
  for (int three_d = 1; three_d >= 1; --three_d)
    for (long span_pos : {8192l})
      for (int depth : {3, 4}) {
        CUtensorMap tm, tm2;
        cuuint32_t estr[3] = {1, 1, 1};
        if (three_d) {
          cuuint64_t dims[3] = {128, (cuuint64_t)H, (cuuint64_t)span_pos};
          cuuint64_t str[2] = {256, (cuuint64_t)H * 256};
          cuuint32_t box[3] = {64, 4, 16};
          enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (char*)buf + (256l << 20), dims, str, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
          cuuint64_t dims[2] = {128, (cuuint64_t)(span_pos * H)};
          cuuint64_t str[1] = {256};
          cuuint32_t box[2] = {64, 64};
          enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        const int tiles = 512;
        const int npt = three_d ? (int)(span_pos / 16) : (int)(span_pos * H / 64 / 2);
        k<<<148, 128, 6 * 32768 + 1024>>>(tm, tm2, three_d, tiles, npt, depth, d_out, mma_mode);
        k<<<148, 128, 6 * 32768 + 1024>>>(tm, tm2, three_d, tiles, npt, depth, d_out, mma_mode);
        if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) { printf("fail\n"); return 1; }
        cudaMemcpy(h.data(), d_out, 148 * 8, cudaMemcpyDeviceToHost);
        double m = 0; for (auto v : h) m += v; m /= 148;
        printf("mma %d %s span %6ld pos (%4ld MB)  depth %d: %7.0f clk per 32 KB tile  (%5.1f B/clk/SM)\n",
               mma_mode, three_d ? "3D {64,4,16}" : "2D {64,64}  ", span_pos, span_pos * H * 256 >> 20, depth,
               m / tiles, 32768.0 * tiles / m);
      }
  return 0;
}
