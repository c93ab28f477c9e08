/* coserve_cuda.h -- C ABI of libcoserve_cuda.so, the B200 (sm_100a) drop-in for the
 * co-serving iteration of FlexLLM (arXiv 2402.18789).
 *
 * The reference (/root/reference/proj) is a header-only C++20 library with no FFI; the
 * entry points below are what a binding of its hot path needs:
 *
 *   cs_engine_create / cs_engine_set_weight  <- TinyModel::init (tiny_model.hpp:44-67):
 *                                               model config + frozen weights + LoRA A,B
 *   cs_step (FT forward window)              <- forward_full (tiny_model.hpp:181-221) executed
 *                                               as forward_window fused with
 *                                               inference prefill/decode rows
 *   cs_step (FT backward window)             <- backward_full (tiny_model.hpp:259-327) executed
 *                                               as backward_window
 *   cs_step_result.ft_loss_sum               <- generative_loss
 *   cs_read_lora_grads                       <- LoraGrads (tiny_model.hpp:71-83)
 *   cs_read_kvgrad                           <- OracleLayerGrads dk/dv (tiny_model.hpp:248-251)
 *   cs_adam_step                             <- Adam once per mini-batch
 *   cs_sched_*                               <- latency / max_finetune_tokens / try_admit /
 *                                               plan_iteration / advance_finetune
 *
 * Conventions (mirroring the reference's):
 *   - every call returns CS_OK (0) or a negative status; the message is in cs_last_error()
 *     (thread-local).  CS_ERR_INVALID_ARGUMENT <-> std::invalid_argument,
 *     CS_ERR_RUNTIME <-> std::runtime_error, CS_ERR_CACHE_DESYNC / CS_ERR_ORDERING are the
 *     spec's cache-desync / ordering-violation errors.
 *   - host buffers passed in are copied; the caller keeps ownership.  The engine owns all
 *     device memory.  One host thread per engine; stream-ordered; not thread-safe.
 *   - weights use the reference layout: row-major [in, out] (x . W convention).
 */
#ifndef COSERVE_CUDA_H
#define COSERVE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 3  /* 2: policy / VTC / tail-control / sim-clock config fields, per-tenant stats, fwd_window_ms; 3: ITL + timed-arrival SLO stats, spatial / isolation policies */

#define CS_OK 0
#define CS_ERR_INVALID_ARGUMENT (-1)
#define CS_ERR_RUNTIME (-2)
#define CS_ERR_CUDA (-3)
#define CS_ERR_CACHE_DESYNC (-4)
#define CS_ERR_ORDERING (-5)
#define CS_ERR_OOM (-6)
#define CS_ERR_NCCL (-7)

const char* cs_last_error(void);
int cs_version(void);
/* debugging: SM-clock event timeline of one CTA of the instrumented kernels */
int64_t cs_debug_trace(int cta, void* dev_buf, int64_t capacity);

/* ---------------------------------------------------------------- primitives (device ptrs) */
/* C[M,N] (op)= A[M,K] . B[N,K]^T, bf16 operands (K contiguous), fp32 accumulate on
 * tcgen05/TMEM.  epi: 0 bf16 store (+bias), 1 fp32 store, 2 fp32 +=, 3 fp32 atomic +=,
 * 5 SwiGLU (B's rows interleaved in 64-row [gate | up] blocks, N % 128 == 0: C (bf16, ldc >= N/2)
 * receives silu(bf16 gate) * bf16 up for N/2 columns and zeros in [N/2, ldc)).
 * bn in {0(auto),16,32,64,128,256}; splits 0 = auto (fp32 epilogues only). */
int cs_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                 int64_t M, int64_t N, int64_t K, int epi, const float* bias, int bn, int splits,
                 void* stream);
/* Same with B stored [K, N] row-major (N contiguous, ldb >= N): the MN-major B operand the
 * engine's backward dX GEMMs use to read the forward weight layout (one copy of the frozen
 * weights serves x.W and dY.W^T).  bn in {0, 64, 128, 256}; no bias. */
int cs_gemm_bf16_mn(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                    int64_t M, int64_t N, int64_t K, int epi, int bn, int splits, void* stream);

/* ---------------------------------------------------------------- engine */
typedef struct cs_model_config {
  int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab, lora_rank;
  int32_t norm;     /* 0 = none (reference TinyModel), 1 = RMSNorm                  */
  int32_t act;      /* 0 = ReLU on up (reference),      1 = SwiGLU (gate || up)      */
  int32_t rope;     /* 0 = none (reference),            1 = rotate-half RoPE         */
  int32_t qkv_bias; /* Qwen-style QKV bias                                          */
  float rope_theta;
  float rms_eps;
  int32_t page_size;  /* tokens per KV page                                         */
  int32_t n_pages;    /* KV pool pages (every layer has its own pool of n_pages)    */
  int32_t max_tokens; /* max tokens in one iteration (inference + FT forward rows)  */
  int32_t max_ft_len; /* max finetuning sequence length L                           */
  int32_t max_segments;
} cs_model_config;

typedef struct cs_engine cs_engine;

/* Tensor parallelism (shard_eval.hpp:111-192 evaluates the same layout):
 * tp_size > 1 shards the q/kv heads and the ffn columns over the ranks (QKV and gate||up
 * column-parallel, O and down row-parallel, LoRA A row-sharded with B replicated and its
 * up-projection folded into the down partial sums); the residual stream is replicated and
 * all-reduced after O and down (forward) and after the gate||up / QKV input-gradient GEMMs
 * (backward window); dB is all-reduced once per mini-batch inside cs_adam_step.
 * Every rank gets the SAME plan.  nccl_unique_id: 128 bytes from cs_nccl_unique_id() on
 * rank 0, shared by the host (one process per GPU).  Weights are passed whole to every rank
 * (reference layout); each engine keeps its shard.  Read-backs (lora, grads, kv, kvgrad) are
 * this rank's shard; grad_b is this rank's partial sum until cs_adam_step. */
int cs_engine_create(const cs_model_config* cfg, int device, int tp_rank, int tp_size,
                     const void* nccl_unique_id, cs_engine** out);
int cs_nccl_unique_id(void* out128);
/* Single-process TP: the ranks are engines of this process (one host thread each, cs_step
 * called concurrently with the same plan); the all-reduce is a one-shot peer kernel over
 * the ranks' buffers (NVLink peer access across devices, or one device for testing). */
typedef struct cs_tp_group cs_tp_group;
int cs_tp_group_create(int tp_size, cs_tp_group** out);
int cs_tp_group_destroy(cs_tp_group* g); /* after every engine of the group is destroyed */
int cs_engine_create_tp_local(const cs_model_config* cfg, int device, int tp_rank,
                              cs_tp_group* group, cs_engine** out);
/* Cross-process peer-memory TP (one process per GPU, no NCCL): create every rank with
 * cs_engine_create_ipc, export each rank's 64-byte CUDA IPC handle of its engine arena with
 * cs_engine_ipc_handle, share them through any host channel (bench.py: torch.distributed),
 * then cs_engine_ipc_attach on every rank with all ranks' handles and arena sizes in rank
 * order ([tp_size][64] bytes, [tp_size] int64).  From then on the row-parallel GEMMs write
 * their partial tiles straight into the owners' staging over NVLink (the fused GEMM +
 * all-reduce of a single-process group) and the remaining all-reduces are one-shot peer
 * kernels; cross-rank ordering is a device-side flag barrier.  Same plan on every rank. */
int cs_engine_create_ipc(const cs_model_config* cfg, int device, int tp_rank, int tp_size,
                         cs_engine** out);
int cs_engine_ipc_handle(cs_engine* e, void* out64, int64_t* arena_bytes);
int cs_engine_ipc_attach(cs_engine* e, const void* handles, const int64_t* arena_bytes);
int cs_engine_destroy(cs_engine* e);
/* dtype: 0 = f64, 1 = f32.  name in {embed, unembed, final_norm, wq, wk, wv, wo, w_gate, w_up,
 * w_down, lora_a, lora_b, bq, bk, bv, norm1, norm2}; shapes in the reference layout. */
int cs_engine_set_weight(cs_engine* e, const char* name, int layer, const void* host, int dtype,
                         int64_t rows, int64_t cols);
/* LoRA A/B master weights (fp32) read back as f64 (e.g. after cs_adam_step). */
int cs_engine_get_lora(cs_engine* e, int layer, double* a_out, double* b_out);
/* Device-side random init with the reference's scales (tiny_model.hpp:51-63) for the
 * performance configs (no parity claim; counter-based RNG). */
int cs_engine_init_random(cs_engine* e, uint64_t seed);

#define CS_SEG_DECODE 0
#define CS_SEG_PREFILL 1
#define CS_SEG_FT_FWD 2

typedef struct cs_segment {
  int32_t kind;      /* CS_SEG_*                                                    */
  int32_t q_start;   /* first row of this segment inside the token batch           */
  int32_t q_len;     /* rows                                                       */
  int32_t ctx_start; /* position of the first row (= tokens already in its cache)  */
  int32_t page_off;  /* offset of its page table inside plan->page_table           */
  int32_t n_pages;   /* pages covering positions [0, ctx_start + q_len)            */
  int32_t sample;    /* 1: return argmax next token of the last row                */
  int32_t adapter;   /* 1: rows pass through the LoRA bypass                        */
} cs_segment;

#define CS_FT_NONE 0
#define CS_FT_FORWARD 1
#define CS_FT_BACKWARD 2

typedef struct cs_ft_window {
  int32_t phase;           /* CS_FT_*                                                */
  int32_t seq_len;         /* L of the finetuning sequence                           */
  int32_t l;               /* forward: l_i (window start); backward: l_j (window end) */
  int32_t s;               /* window tokens                                          */
  int32_t layer;           /* backward: layer n                                      */
  const int32_t* targets;  /* forward: next-token ids of the s rows (-1 = none)      */
  int32_t page_off;        /* FT sequence page table inside plan->page_table         */
  int32_t n_pages;
} cs_ft_window;

typedef struct cs_iteration_plan {
  int32_t n_tokens;
  const int32_t* tokens; /* [n_tokens]; FT forward rows (if any) are the last segment */
  int32_t n_segments;
  const cs_segment* segments;
  const int32_t* page_table;
  int32_t page_table_len;
  cs_ft_window ft;
  /* further backward windows run after `ft` in this iteration, in order (each must continue
   * Alg. 2's descending order; they may cross into the next lower layer) */
  int32_t n_extra_bwd;
  const cs_ft_window* extra_bwd;
} cs_iteration_plan;

typedef struct cs_step_result {
  int32_t* next_tokens;  /* [n_segments] or NULL; -1 for unsampled segments           */
  float* logits;         /* [n_sampled, vocab] or NULL                                */
  double ft_loss_sum;    /* summed next-token CE of this forward window               */
  float iteration_ms;    /* device time of the step (CUDA events)                     */
} cs_step_result;

int cs_step(cs_engine* e, const cs_iteration_plan* plan, cs_step_result* result);
/* Asynchronous variant: enqueue only (no host sync, no read-back); pair with cs_sync. */
int cs_step_async(cs_engine* e, const cs_iteration_plan* plan);
int cs_sync(cs_engine* e, cs_step_result* result);

int cs_adam_step(cs_engine* e, float lr, float beta1, float beta2, float eps);
int cs_zero_lora_grads(cs_engine* e);
/* abandon the active finetuning mini-batch (cache length 0, backward state cleared, grads 0) */
int cs_engine_reset_ft(cs_engine* e);
int cs_read_lora_grads(cs_engine* e, int layer, double* grad_a, double* grad_b);
/* dK, dV accumulated (ΔKVAccum) for the layer currently being back-propagated, rows [0, L). */
int cs_read_kvgrad(cs_engine* e, int32_t L, double* dk_out, double* dv_out);
/* K/V of one sequence (by page table) at one layer, positions [0, len): [len, kv_dim]. */
int cs_read_kv(cs_engine* e, int layer, const int32_t* pages, int32_t len, double* k_out,
               double* v_out);
/* dLoss/d(input of layer) rows [0, L) produced by the last backward windows. */
int cs_read_dy(cs_engine* e, int32_t L, double* out);

/* Allocation audit (Matrix::alloc_hook, matrix.hpp:16-25): hook(name, elements, elem_bytes)
 * once per device buffer of the engine's arena (everything is carved at create time: steps
 * allocate nothing); transient_allocs = device allocations made outside the arena so far
 * (weight-upload staging only). */
typedef void (*cs_alloc_hook)(const char* name, int64_t elems, int32_t elem_bytes, void* user);
int cs_engine_alloc_audit(cs_engine* e, cs_alloc_hook hook, void* user, int64_t* transient_allocs);

/* ---------------------------------------------------------------- host scheduler (no GPU) */
typedef struct cs_latency_profile {
  double t0_ms;
  double slope_ms_per_token;
  double knee_tokens;      /* <= 0 -> infinite knee                                   */
  double bwd_token_weight; /* cost of a backward-window token in forward tokens; <= 0 -> 1 */
  double attn_fwd_ms_per_token_ctx; /* forward window extra: a_f * s * (l + s/2)         */
  double attn_bwd_ms_per_token_ctx; /* backward window extra: a_b * s * (l_j - s/2)      */
  double bwd_layer0_weight;  /* layer-0 (pruned) backward window cost factor; <= 0 -> 1     */
  double decode_ms_per_row;    /* inference decode row slope; <= 0 -> slope_ms_per_token     */
  double prefill_ms_per_token; /* inference prefill token slope; <= 0 -> slope_ms_per_token  */
  double fwd_window_ms;        /* fixed cost of a finetuning forward window; <= 0 -> none     */
} cs_latency_profile;

double cs_sched_latency(const cs_latency_profile* p, int64_t c, int64_t s);
int64_t cs_sched_max_finetune_tokens(const cs_latency_profile* p, int64_t c, double slo_ms);

/* ---------------------------------------------------------------- co-serving loop */
/* One run of the co-serving engine loop over synthetic arrivals:
 * plan_iteration -> cs_step -> advance state -> Adam per mini-batch.  engine == NULL runs the
 * same loop on a simulated clock (predicted latency): plans are then
 * bit-reproducible and are what the scheduler parity tests compare against the oracle. */
typedef struct cs_coserve_config {
  double rate_rps, duration_s, burst_amplitude, burst_period_s;
  double tpot_slo_ms, ttft_slo_ms, budget_ms;
  int32_t max_batch, chunk_size, max_tokens, max_ft_window;
  cs_latency_profile profile;
  int32_t ft_seq_len, growth_tokens, warmup_iters, timed_iters, prepopulate, adaptive;
  int32_t profile_timed; /* switch on cs_engine_set_profiling at the first timed iteration */
  int32_t multi_layer_bwd; /* one iteration may carry backward windows of several layers     */
  uint64_t seed;
  /* simulation-only (engine == NULL): model depth, vocab and KV pool */
  int32_t n_layers, vocab, page_size;
  int64_t total_pages;
  /* scheduling policy (§8.2): 0 co-serving, 1 temporal sharing with a fixed
   * inference frequency temporal_n, 2 dynamic temporal sharing */
  int32_t policy, temporal_n;
  /* 1: advance the loop clock by the planner's predicted latency even with an engine (a
   * timing-independent plan sequence, e.g. for profiling runs under ncu) */
  int32_t sim_clock;
  /* Virtual Token Counter fair admission (Appendix C): vtc = 1 enables it; arrivals
   * go to tenant 0 with probability tenant0_share, else uniformly to 1..n_tenants-1; charges
   * w_p per prompt token at admission, w_q per generated token, w_r per finetuning token to
   * ft_tenant (-1: nobody) */
  int32_t vtc, n_tenants, ft_tenant;
  double tenant0_share, vtc_wp, vtc_wq, vtc_wr;
  /* tail control (adaptive runs; 0 = off): planner budget = tail_target x TPOT SLO / q95 of
   * the recent measured/predicted iteration-time ratios */
  double tail_target;
  /* policy 3 spatial sharing / 4 resource isolation: inference fraction
   * spatial_rho in (0, 1), interference spatial_gamma >= 1 (< 1 -> 1.15; isolation: 1) */
  double spatial_rho, spatial_gamma;
} cs_coserve_config;

typedef struct cs_coserve_stats {
  int64_t iters;
  double timed_ms, timed_device_ms;
  int64_t ft_fwd_tokens, ft_bwd_tokens;
  double ft_fwd_ms, ft_bwd_ms;
  int64_t minibatches_done;
  int64_t inf_tokens, gen_tokens, requests_done, requests_slo_ok, evictions;
  double ttft_p50_ms, ttft_p99_ms, tpot_p50_ms, tpot_p99_ms;
  double iter_p50_ms, iter_p99_ms, iter_max_ms; /* timed iterations with inference work */
  int64_t gpu_launches;                        /* kernels launched in the timed region   */
  int64_t h2d_bytes, d2h_bytes;                /* host<->device bytes in the timed region */
  /* VTC (tenants 0..7): cumulative weighted service, completed requests, max spread of the
   * backlogged tenants' counters (Lemma 1), max |W_0 - W_1| over intervals where tenants 0
   * and 1 are both backlogged (Theorem 1) */
  double tenant_service[8];
  int64_t tenant_done[8];
  double vtc_spread_max, vtc_pair_gap_max;
  /* observable in short runs: inter-token latency over every decoding request in the timed
   * region; requests that arrived in the timed region: count, completed, completed inside both
   * SLOs, unfinished with a first-token wait already past the TTFT SLO (misses) */
  double itl_p50_ms, itl_p99_ms, itl_max_ms;
  int64_t itl_samples;
  int64_t timed_arrivals, timed_done, timed_slo_ok, timed_unfinished_miss;
} cs_coserve_stats;

typedef struct cs_iter_log {
  double t_ms, pred_ms, ms, device_ms;
  int32_t c, s, phase, layer, l, n_decode, n_prefill, n_running, n_queue, timed;
} cs_iter_log;

int cs_coserve_run(cs_engine* e, const cs_coserve_config* cfg, cs_coserve_stats* stats,
                   cs_iter_log* log, int64_t log_cap, int64_t* log_len);
/* kernels launched by this library so far (the driver's gpu_launches claim) */
int64_t cs_engine_launch_count(cs_engine* e);
/* Live profiling: when on, every GEMM / attention launch is bracketed by CUDA events on the
 * engine stream; cs_engine_read_profile returns the summed device ms, algorithmic FLOPs and
 * bytes and launch count per kind (0 = tcgen05 GEMM, 1 = attention fwd bandwidth kernel
 * (decode rows, incl. the split-KV combine), 2 = attention bwd, 3 = attention fwd tcgen05
 * kernel (prefill / FT rows), 4 = TP all-reduce, 5 = the decode kernel alone)
 * since profiling was switched on. */
int cs_engine_set_profiling(cs_engine* e, int on);
int cs_engine_read_profile(cs_engine* e, int kind, double* ms, double* flops, double* bytes,
                           int64_t* launches);
/* Max over the engine's TP group of n <= 8 host doubles, in place, identical on every rank
 * (no-op at tp_size 1; every rank calls it, like cs_step).  cs_coserve_run uses it so the
 * per-rank loops of one TP group see the same clock and plan the same iterations. */
int cs_engine_tp_sync_max(cs_engine* e, double* vals, int n);
/* model depth, vocab and KV pool geometry of an engine */
int cs_engine_pool_info(cs_engine* e, int32_t* n_layers, int32_t* vocab, int32_t* page_size,
                        int64_t* n_pages);

#ifdef __cplusplus
}
#endif
#endif /* COSERVE_CUDA_H */
