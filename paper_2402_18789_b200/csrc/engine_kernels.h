// engine_kernels.h -- parameter blocks + launchers of the non-GEMM kernels of the step.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cuda.h>

namespace cs {

using bf16 = __nv_bfloat16;

// ------------------------------------------------------------------ attention
struct AttnSeg {
  int q_start, q_len, ctx_start, page_off;
};

struct AttnWork {  // one CTA of attn_fwd_kernel
  int seg, q0, nq, kv_head, k_begin, k_end, part, pad;
};

// one decode work item (attn_decode_swap / _stream kernels): the segment fields and the KV-pool rows of the first 8
// 16-key boxes are resolved on the host, so the kernel's prologue is one load deep (work item
// -> TMA issue / Q loads) instead of three (work -> segment -> page table -> TMA)
struct AttnDecWork {
  int q_row, pos0, page_off, kv_head, k_begin, k_end, part, nq;
  int prow[8];
};

struct AttnCombine {  // one CTA of attn_combine_kernel
  int seg, q0, nq, kv_head, part0, n_parts, pad0, pad1;
};

struct AttnFwdParams {
  const bf16* q;
  long q_ld;
  const bf16* k_pool;
  const bf16* v_pool;
  int kv_dim, page_size;
  const int* page_table;
  const AttnSeg* segs;
  const AttnWork* work;
  const AttnDecWork* dwork;  // decode kernels only
  const AttnCombine* combine;
  bf16* out;
  long out_ld;
  float* lse;
  int lse_ld;
  float* part_o;
  float* part_lse;
  int grp;
  float scale_log2;
  int part_rows = 64;  // rows per split-KV part in part_o / part_lse (combine)
  int comb_slices = 4;  // attn_fwd's combine grid.y: 16-row slices of the largest item
  int max_dec_rows = 16;  // attn_decode: max packed rows (q_len x group) over the work items
};

struct AttnBwdParams {
  const bf16* q_cache;  // [L][q_ld] roped Q of the FT sequence (this layer)
  long q_ld;
  const bf16* dO;       // [b-a][do_ld]
  long do_ld;
  const bf16* O;        // saved attention output rows [a,b) [b-a][o_ld]
  long o_ld;
  const float* lse;     // [L][lse_ld]
  int lse_ld;
  float* delta;         // [b-a][delta_ld]
  int delta_ld;
  const bf16* k_pool;
  const bf16* v_pool;
  int kv_dim, page_size;
  const int* page_table;
  int page_off;
  int a, b;
  float* dq;            // [b-a][dq_ld]
  long dq_ld;
  float* dk_acc;        // ΔKVAccum [L][acc_ld]
  float* dv_acc;
  long acc_ld;
  int grp;
  float scale, scale_log2;
  int tiles_per_cta = 1 << 30;  // fused kernel: query tiles per CTA (set by attn_bwd_fused)
};

// decode rows (q_len * group <= 16): HBM-bound paged kernel (attn_decode.cu); run before
// attn_fwd, whose combine pass also merges the decode partials
cudaError_t attn_decode(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                        int head_dim, int n_work, cudaStream_t st);
// keys per warp tile, warps per decode CTA, resident CTAs per SM and whether the variant is
// the persistent per-warp stream kernel (one warp per item) -- the host work split follows it
void attn_decode_geometry(int head_dim, int* keys_per_tile, int* nwarp, int* ctas_per_sm,
                          int* streams);
// merge split-KV partials listed in p.combine (p.part_rows rows per part)
cudaError_t attn_combine(const AttnFwdParams& p, int head_dim, int n_combine, cudaStream_t st);
cudaError_t attn_fwd(const AttnFwdParams& p, int head_dim, int n_work, int n_combine,
                     cudaStream_t st);
cudaError_t attn_bwd(const AttnBwdParams& p, int head_dim, int n_heads, cudaStream_t st);
void attn_bwd_delta_kernel_launch(const AttnBwdParams& p, int rows, int n_heads, cudaStream_t st);
// fused tcgen05 backward (head_dim 128, GQA group <= 8): dK / dV into ΔKVAccum and dQ (fp32,
// zeroed here, then reduce-added per (key block, query tile) through tmDQ: {128 d, Hq, rows}
// fp32, box {64, grp, 64 / grp})
cudaError_t attn_bwd_fused(const AttnBwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                           const CUtensorMap& tmK128, const CUtensorMap& tmV128, const CUtensorMap& tmQ3,
                           const CUtensorMap& tmO3, const CUtensorMap& tmDQ, int n_heads, cudaStream_t st);
// tcgen05 forward for prefill / finetuning-window tiles (head_dim 128): two 128-row query tiles
// per CTA (work items of 2 * (128 / group) positions), P kept in TMEM
cudaError_t attn_fwd_tc2(const AttnFwdParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                         const CUtensorMap& tmK128, const CUtensorMap& tmV128, int n_work,
                         cudaStream_t st);

// ------------------------------------------------------------------ elementwise (elem.cu)
void embed_gather(const int* tokens, const bf16* embed, float* x, int T, int h, cudaStream_t st);

// out_bf16[r] = bf16(norm ? x*rstd*g : x); rstd_out optional
void rmsnorm_cast(const float* x, long ldx, const float* g, bf16* out, long ldo, float* rstd_out,
                  int rows, int h, float eps, int use_norm, cudaStream_t st);
// rows gathered by index (sampling / head rows)
void rmsnorm_cast_gather(const float* x, long ldx, const int* idx, const float* g, bf16* out,
                         long ldo, float* rstd_out, int rows, int h, float eps, int use_norm,
                         cudaStream_t st);

struct RopeAppendParams {
  bf16* qkv;
  long ld;
  const int* row_pos;    // [T] absolute position
  const int* row_seg;    // [T] segment index
  const AttnSeg* segs;
  const int* page_table;
  bf16* k_pool;
  bf16* v_pool;
  int page_size;
  int n_heads, n_kv_heads, head_dim;
  int use_rope;
  float rope_theta;
  int T;
  int ft_row0;           // rows >= ft_row0 are finetuning forward rows (or T)
  bf16* q_cache;         // [L][q_dim] (this layer) or null
};
void rope_append(const RopeAppendParams& p, cudaStream_t st);
// [max_pos][head_dim/2] (cos, sin) table used by rope_append / rope_bwd_pack
void set_rope_table(const float2* tab);

// m[:, :f] = act(gu); m[:, f:ldm] = 0
void act_fwd(const bf16* gu, long ld_gu, bf16* m, long ldm, int rows, int f, int swiglu,
             cudaStream_t st);
// m[row, f + j] = bf16(lu[row - 0, j]) for the adapter rows
void lora_pack(const float* lu, int r, bf16* m, long ldm, int f, int rows, cudaStream_t st);

// scratch: rows * 16 keys
void argmax_rows(const float* logits, long ld, int rows, int V, int* out,
                 unsigned long long* scratch, cudaStream_t st);

// Fused CE over a chunk of logits rows: loss[i] = lse - logit[t]; dlogits = (softmax - onehot)
// * inv_norm (rows with target < 0 -> 0 loss, 0 grad)
void ce_fwd_bwd(const float* logits, long ld, const int* targets, int rows, int V,
                float inv_norm, float* loss, bf16* dlogits, long ldd, cudaStream_t st);

// out = resid + (norm ? rms_bwd(x, g, rstd, dh) : dh); optional bf16 copy
void rms_bwd_add(const float* resid, long ldr, const float* x, long ldx, const float* g,
                 const float* rstd, const float* dh, long ldh, float* out, long ldo,
                 bf16* out_b, long ldob, int rows, int h, int use_norm, cudaStream_t st);

// MLP + LoRA-A backward: dgu (bf16) from dm, saved gu/m; dA[f,r] += m^T dlu
void mlp_bwd(const bf16* dm, long ld_dm, const bf16* saved, long ld_s, const float* dlu, int r,
             bf16* dgu, long ld_dgu, float* dA, int rows, int f, int swiglu, cudaStream_t st);

// dB += lu^T dY, and dycat[:, :h] = bf16(dY) in the same pass (dlu = dY B^T is then a tcgen05
// GEMM over dycat, packed into its LoRA columns by lora_pack)
void lora_db(const float* dY, long ldy, const float* lu, int r, int rows, int h, float* dB,
             bf16* dycat, long ldc, cudaStream_t st);

// dqkv = [rope^-1(dq) | rope^-1(dk_acc[a:b]) | dv_acc[a:b]] (bf16)
void rope_bwd_pack(const float* dq, long ldq, const float* dk, const float* dv, long ld_acc,
                   int a, int rows, int n_heads, int n_kv_heads, int head_dim, int use_rope,
                   float theta, bf16* out, long ldo, cudaStream_t st);

struct AdamParams {
  float* A;   // [n_layers][f][r] fp32 master
  float* B;   // [n_layers][r][h]
  const float* gA;
  const float* gB;
  float* mA;
  float* vA;
  float* mB;
  float* vB;
  bf16* A_t;        // [n_layers][16][f]          (lu GEMM B operand)
  bf16* B_t;        // [n_layers][16][h]          (dlu GEMM B operand)
  bf16* down_cat;   // [n_layers][down_rows][f + 64]  rows < h: cols f.. = B^T; rows h.. = A^T
  int down_rows;    // h + 64: A^T rides in down_cat (the MN-major backward operand)
  int n_layers, f, r, h;
  float lr, b1, b2, eps, bc1, bc2;
};
void adam_step(const AdamParams& p, int update, cudaStream_t st);

// weight prep: dst_bf16 (optionally transposed) from fp32 staging; dst[i*ldd + j]
void cast_f32_bf16(const float* src, int rows, int cols, bf16* dst, long ldd, int transpose,
                   cudaStream_t st);
// transposed cast into 64-row blocks: dst row (c / 64) * blk_stride + blk_off + c % 64
void cast_f32_bf16_interleaved(const float* src, int rows, int cols, bf16* dst, long ldd, int blk_stride,
                               int blk_off, cudaStream_t st);
void init_normal_bf16(bf16* dst, long n, float scale, uint64_t seed, cudaStream_t st);
void init_normal_f32(float* dst, long n, float scale, uint64_t seed, cudaStream_t st);
void fill_f32(float* dst, long n, float v, cudaStream_t st);

}  // namespace cs
