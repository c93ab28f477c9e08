// kernels.h -- host-side launchers of the sm_100a kernels (internal to libcoserve_cuda.so).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cuda.h>

#include <atomic>

namespace cs {

extern std::atomic<long> g_launches;  // kernels launched by this library (process-wide)

// Launch with programmatic stream serialization (PDL): the kernel's prologue overlaps the
// previous kernel's tail; the kernel must call griddep_wait() before touching shared data.
// CS_PDL=0 disables it (plain stream order).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------------------ GEMM (gemm.cu)
enum GemmEpi : int {
  EPI_BF16 = 0,        // C_bf16 = acc (+ bias)
  EPI_F32 = 1,         // C_f32  = acc
  EPI_F32_ADD = 2,     // C_f32 += acc   (residual stream; split-K via atomics)
  EPI_F32_ATOMIC = 3,  // C_f32 += acc with atomics (caller-initialised C)
  EPI_F32_SCATTER = 4, // row-parallel TP partial -> the owning rank's staging slot (GemmScatter)
  // gate||up projection with the SwiGLU fused into the epilogue: B's rows (the weights) are
  // interleaved in 64-row blocks [gate 64b..64b+63 | up 64b..64b+63], so every 128-column group
  // of the output holds matching gate / up columns.  C (bf16, ldc) receives
  // m[:, j] = silu(bf16(g_j)) * bf16(u_j) for j < m_cols and zeros in [m_cols, ldc); rows >=
  // c2_row0 also store the raw bf16 gate / up (interleaved layout) to C2 + (row - c2_row0) * ldc2
  // (the finetuning rows' saved activations).  BN >= 128, no K split.
  EPI_SWIGLU = 5,
  // QKV projection with RoPE and the KV-cache append fused into the epilogue (head_dim 128;
  // QkvEpi): C (bf16 [T, q|k|v], +bias) receives the roped q heads (and the FT rows' copy in
  // q_cache); the roped k and the v heads go straight to the row's paged K / V slot.  Rounding
  // points as rope_append after a bf16 GEMM: bf16(acc + bias), rotation in fp32, bf16.
  EPI_QKV_ROPE = 6,
};

struct QkvEpi {
  const int* row_pos = nullptr;    // [T] absolute position
  const int* row_slot = nullptr;   // [T] KV-pool row (page * page_size + pos % page_size)
  __nv_bfloat16* k_pool = nullptr;
  __nv_bfloat16* v_pool = nullptr;
  __nv_bfloat16* q_cache = nullptr;  // [L][q_dim] (this layer) or null
  const float2* rope_tab = nullptr;  // [max_pos][64] (cos, sin)
  int q_dim = 0, kv_dim = 0, ft_row0 = 0, use_rope = 0;
};

// EPI_F32_SCATTER: output row `row` belongs to rank owner = row / rows_per_owner; the fp32
// partial goes to peer[owner] + ((rank * rows_per_owner) + row - owner * rows_per_owner) * ldc,
// i.e. slot `rank` of the owner's [ranks][rows_per_owner][ldc] staging buffer (peer memory over
// NVLink / NVSwitch; plain stores, or fp32 atomics into the zeroed slot for split-K).
struct GemmScatter {
  float* peer[8] = {};
  int rows_per_owner = 0;
  int rank = 0;
};

struct GemmDesc {
  const void* A = nullptr;  // bf16 [M, K] row-major, leading dim lda (elements)
  long lda = 0;
  long a_rows = 0;          // rows described by the TMA map (>= M; 0 -> M)
  const void* B = nullptr;  // bf16 [N, K] row-major, leading dim ldb
  long ldb = 0;
  long b_rows = 0;          // (>= N; 0 -> N)
  void* C = nullptr;
  long ldc = 0;
  long M = 0, N = 0, K = 0;
  int epi = EPI_BF16;
  const float* bias = nullptr;  // [N] (EPI_BF16 only)
  int bn = 0;                   // 0 = heuristic
  int splits = 0;               // 0 = heuristic (fp32 epilogues only)
  int max_ctas = 0;             // 0 = #SMs
  int b_const = 0;              // B not produced by the preceding kernel (weights): PDL prefetch
  GemmScatter scatter;          // EPI_F32_SCATTER only
  int b_mn = 0;                 // 1: B stored [K rows][N cols] (ldb >= N): MN-major operand
  void* C2 = nullptr;           // EPI_SWIGLU: saved gate / up rows (see above)
  long ldc2 = 0;
  int c2_row0 = 0;
  int m_cols = 0;               // EPI_SWIGLU: width of m (the ffn size f)
  QkvEpi qkv;                   // EPI_QKV_ROPE
};

cudaError_t gemm_tn(const GemmDesc& d, cudaStream_t st);
// cached 2D bf16 TMA map (SWIZZLE_128B, box = 64 columns x box_rows rows); 0 on success
int make_map(CUtensorMap* out, const void* ptr, long rows, long cols, long ld, int box_rows);
// 3D bf16 map {d0 (contiguous), d1, d2}, SWIZZLE_128B, box {64, box1, box2}
int make_map_3d(CUtensorMap* out, const void* ptr, long d0, long d1, long d2, long stride1_bytes,
                long stride2_bytes, int box1, int box2);
int make_map_3d_plain(CUtensorMap* out, const void* ptr, long d0, long d1, long d2, long stride1_bytes,
                      long stride2_bytes, int box0, int box1, int box2);
// 3D fp32 map without swizzle (bulk tensor reduce-add targets), box = {box0, box1, box2}
int make_map_3d_f32(CUtensorMap* out, const void* ptr, long d0, long d1, long d2, long stride1_bytes,
                    long stride2_bytes, int box0, int box1, int box2);
int gemm_pick_bn(long M, long N);

}  // namespace cs
