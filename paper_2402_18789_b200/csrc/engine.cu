// engine.cu -- the co-serving engine behind the C ABI (include/coserve_cuda.h).
//
// One cs_step runs one iteration of FlexLLM's co-serving loop (SPEC.md:687-690 step 3):
//   * forward over the concatenated token batch [decode rows | prefill-chunk rows | FT
//     forward-window rows] through the shared frozen weights: every GEMM is
//     one tcgen05 launch over all rows; attention is one launch over all segments; the LoRA
//     bypass applies to the adapter-row suffix only (segmented, K-concatenated into the
//     down projection); FT rows save only what survives graph pruning and
//     fold the loss-head gradient (loss_head_grad, tiny_model.hpp:223-246) in immediately.
//   * optionally one token-level backward window at layer n (Alg. 2 lines 14-21):
//     rows [l_j - s_j, l_j), ΔKVAccum accumulation, LoRA grads, dX for layer n-1.  Layer 0
//     is pruned to its MLP/LoRA part (no frozen-weight gradients, no dX below).
// Device memory is one arena carved at create time (weights, paged KV pools, FT saved
// activations, scratch sized for max_tokens).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <functional>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "coserve_cuda.h"
#include "engine_kernels.h"
#include "kernels.h"

namespace cs {
int set_error(int code, const std::string& msg);
}

using cs::bf16;

#define CS_CUDA_TRY(x)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (x);                                                                   \
    if (_e != cudaSuccess)                                                                  \
      return cs::set_error(CS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e));   \
  } while (0)

struct cs_engine {
  cs_model_config cfg{};
  int device = 0;
  int tp_rank = 0, tp_size = 1;
  cs::Comm* comm = nullptr;  // tp_size > 1: all-reduce of the row-parallel partial sums
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // decode / small-segment attention on a side stream next to the tcgen05 FT-window attention
  // (forward(): fork after the QKV projection, join before the O projection)
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // dims (per rank: heads and ffn columns are this rank's shard; *_g = whole model)
  int Hq_g, Hkv_g, f_g;
  int h, Hq, Hkv, d, q_dim, kv_dim, nqkv, f, V, r, NL, P, npages, gu_n, f_cat, h_cat, grp;
  int T_max, L_max, S_max, max_seg, head_chunk, max_pos;
  bool swiglu, norm, rope;
  bool use_tc_attn = true;  // CS_ATTN_TC=0 forces the mma.sync path (A/B testing)
  bool use_dec_attn = true;  // CS_ATTN_DEC=0 sends decode rows to the mma.sync tile kernel
  // dX GEMMs read the forward weight layout as an MN-major B operand: one copy of the frozen
  // QKV / O / gate||up / unembedding weights serves x W and dY W^T
  int down_rows = 0;  // per-layer rows of down_cat: h + 64 LoRA-A^T rows (MN-major dm operand)
  // arena (+ the allocation audit of every buffer carved from it, cf. Matrix::alloc_hook)
  struct AuditRec {
    const char* name;
    long elems;
    int elem_bytes;
  };
  std::vector<AuditRec> audit;
  long transient_allocs = 0;  // device allocations outside the arena (weight upload staging)
  uint8_t* arena = nullptr;
  size_t arena_bytes = 0, arena_used = 0;
  // weights
  bf16 *embed, *unembed_t, *unembed;
  float* gf;
  bf16 *wqkv_t, *wo_t, *wgu_t, *down_cat, *A_t, *B_t;
  float *bqkv, *g1, *g2;
  float *loraA, *loraB, *gA, *gB, *mA, *vA, *mB, *vB;
  // KV
  bf16 *k_pool, *v_pool;
  // FT saved (per layer, by position)
  bf16 *ft_q, *ft_o, *ft_gu;
  float *ft_lse, *ft_x, *ft_r1, *ft_rstd1, *ft_rstd2, *ft_lu;
  float *dk_acc, *dv_acc, *dy[2];
  // forward scratch
  float *x, *rstd, *lu, *lse;
  bf16 *xb, *qkv, *attn, *gu, *m;
  bf16* hf;
  float *logits, *dh, *loss_rows, *hrstd;
  bf16* dlog;
  float* samp_logits;
  int* next_tok;
  unsigned long long* amax_part;
  float *part_o, *part_lse;
  float *part_o_tc, *part_lse_tc;  // split-KV parts of the tcgen05 forward (its own stream)
  float* tp_sync;  // [8 ranks][8 values]: cs_engine_tp_sync_max
  // fused row-parallel GEMM + all-reduce (peer-memory groups): staging [ranks][rpo][h] fp32,
  // zero between uses; peer tables exchanged lazily (same call order on every rank)
  float* tp_stage = nullptr;
  bool tp_fused = false;
  bool tp_fused_allowed = true;  // CS_TP_FUSED=0 -> GEMM + separate all-reduce (A/B)
  unsigned* ipc_flags = nullptr;  // IPC groups: [8] barrier slots, one per peer rank
  float* stage_tab[8] = {};
  std::vector<std::pair<void*, std::vector<float*>>> dst_tabs;
  // backward scratch
  bf16 *dycat, *dgu, *dr1b, *dO, *dqkv, *dm;  // dm: dLoss/d(MLP activation), bf16 like dgu
  float *dlu, *dh2, *dr1, *delta, *dq, *dh1;
  float2* rope_tab;
  // per-step upload
  uint8_t* d_meta = nullptr;
  uint8_t* h_meta = nullptr;
  size_t meta_bytes = 0;
  float* h_loss = nullptr;  // pinned [L_max]: the FT window's per-row losses (async D2H)
  int h_loss_n = 0;
  // FT state machine
  int ft_len = 0;          // QKV cache length (forward progress)
  int ft_L = 0;            // sequence length of the active mini-batch
  int bwd_layer = -2;      // -2: not started; n: current layer; -1: done
  int bwd_next_end = 0;    // expected l_j of the next window
  int dy_cur = 0;
  int adam_t = 0;
  // device-side counters
  long launches = 0;
  // live profiling (cs_engine_set_profiling): CUDA events around each GEMM / attention launch
  bool profiling = false;
  struct ProfRec {
    cudaEvent_t a, b;
    double flops, bytes;
    int kind;  // see prof_ms
    long m = 0, n = 0, k = 0;  // GEMM shape (CS_PROF_LOG)
    int epi = -1;
  };
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<ProfRec> recs;
  // kinds: 0 tcgen05 GEMM, 1 attention fwd (bandwidth kernel: decode), 2 attention bwd,
  //        3 attention fwd (tcgen05 kernel: prefill / FT windows), 4 TP all-reduce
  static constexpr int kKinds = 6;  // 5: the decode kernel alone (kind 1 minus combine / gaps)
  double prof_ms[kKinds] = {}, prof_flops[kKinds] = {}, prof_bytes[kKinds] = {};
  long prof_n[kKinds] = {};
  double step_attn_flops = 0, step_attn_bytes = 0, step_tc_flops = 0, step_tc_bytes = 0;
};

namespace {
cudaEvent_t prof_event(cs_engine* e) {
  if (e->ev_used == e->ev_pool.size()) {
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    e->ev_pool.push_back(ev);
  }
  return e->ev_pool[e->ev_used++];
}
void prof_begin(cs_engine* e, cs_engine::ProfRec& r) {
  r.a = prof_event(e);
  r.b = prof_event(e);
  cudaEventRecord(r.a, e->st);
}
void prof_end(cs_engine* e, cs_engine::ProfRec& r) {
  cudaEventRecord(r.b, e->st);
  e->recs.push_back(r);
}
void prof_collect(cs_engine* e) {
  static FILE* plog = [] {  // CS_PROF_LOG=<file>: one line per profiled launch (kind flops bytes ms)
    const char* v = std::getenv("CS_PROF_LOG");
    return v ? std::fopen(v, "w") : nullptr;
  }();
  for (auto& r : e->recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (plog) std::fprintf(plog, "%d %.6g %.6g %.6f %ld %ld %ld %d\n", r.kind, r.flops, r.bytes, ms, r.m, r.n, r.k, r.epi);
    e->prof_ms[r.kind] += ms;
    e->prof_flops[r.kind] += r.flops;
    e->prof_bytes[r.kind] += r.bytes;
    e->prof_n[r.kind] += 1;
  }
  e->recs.clear();
  e->ev_used = 0;
}
}  // namespace

namespace {

template <typename T>
T* carve(cs_engine* e, size_t count) {
  size_t bytes = ((count * sizeof(T)) + 255) & ~size_t(255);
  T* p = reinterpret_cast<T*>(e->arena + e->arena_used);
  e->arena_used += bytes;
  return p;
}

// two-pass carve: first pass measures (arena == nullptr -> counts only)
struct Planner {
  size_t used = 0;
  template <typename T>
  void add(size_t count) { used += ((count * sizeof(T)) + 255) & ~size_t(255); }
};

void layout(cs_engine* e, bool measure, size_t* total) {
  Planner pl;
  auto A = [&](auto** ptr, size_t count, const char* name) {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(*ptr)>>;
    if (measure) {
      pl.add<T>(count);
    } else {
      *ptr = carve<T>(e, count);
      e->audit.push_back({name, (long)count, (int)sizeof(T)});
    }
  };
#define AL(field, count) A(&e->field, (count), #field)
  const size_t NL = e->NL, h = e->h, V = e->V, f = e->f, r = e->r;
  const size_t T = e->T_max, Lm = e->L_max, S = e->S_max;
  AL(embed, V * h);
  AL(unembed_t, V * h);
  AL(gf, h);
  AL(wqkv_t, NL * e->nqkv * h);
  AL(wo_t, NL * h * e->q_dim);
  AL(wgu_t, NL * e->gu_n * h);
  AL(down_cat, NL * e->down_rows * e->f_cat);
  AL(A_t, NL * 16 * f);
  AL(B_t, NL * 16 * h);
  AL(bqkv, NL * e->nqkv);
  AL(g1, NL * h);
  AL(g2, NL * h);
  AL(loraA, NL * f * r);
  AL(loraB, NL * r * h);
  AL(gA, NL * f * r);
  AL(gB, NL * r * h);
  AL(mA, NL * f * r);
  AL(vA, NL * f * r);
  AL(mB, NL * r * h);
  AL(vB, NL * r * h);
  const size_t kv = NL * (size_t)e->npages * e->P * e->kv_dim;
  AL(k_pool, kv);
  AL(v_pool, kv);
  AL(ft_q, NL * Lm * e->q_dim);
  AL(ft_o, NL * Lm * e->q_dim);
  AL(ft_gu, NL * Lm * e->gu_n);
  AL(ft_lse, NL * Lm * e->Hq);
  AL(ft_x, e->norm ? NL * Lm * h : 1);
  AL(ft_r1, e->norm ? NL * Lm * h : 1);
  AL(ft_rstd1, NL * Lm);
  AL(ft_rstd2, NL * Lm);
  AL(ft_lu, NL * Lm * r);
  AL(dk_acc, Lm * e->kv_dim);
  AL(dv_acc, Lm * e->kv_dim);
  AL(dy[0], Lm * h);
  AL(dy[1], Lm * h);
  AL(x, T * h);
  AL(rstd, T);
  AL(lu, T * r);
  AL(lse, T * e->Hq);
  AL(xb, T * h);
  AL(qkv, T * e->nqkv);
  AL(attn, T * e->q_dim);
  AL(gu, T * e->gu_n);
  AL(m, T * e->f_cat);
  const size_t C = e->head_chunk;
  AL(hf, std::max(C, (size_t)e->max_seg) * h);
  AL(logits, std::max(C, (size_t)e->max_seg) * V);
  AL(dlog, C * V);
  AL(dh, C * h);
  AL(hrstd, C);
  AL(loss_rows, Lm);
  AL(samp_logits, (size_t)e->max_seg * V);
  AL(next_tok, e->max_seg);
  AL(amax_part, (size_t)e->max_seg * 16);
  const size_t max_parts = 4096;
  AL(part_o, max_parts * 64 * e->d);
  AL(part_lse, max_parts * 64);
  AL(part_o_tc, max_parts * 64 * e->d);
  AL(part_lse_tc, max_parts * 64);
  AL(dycat, S * e->h_cat);
  AL(dgu, S * e->gu_n);
  AL(dr1b, S * h);
  AL(dO, S * e->q_dim);
  AL(dqkv, S * e->nqkv);
  AL(dlu, S * r);
  AL(dm, S * f);
  AL(dh2, S * h);
  AL(dr1, S * h);
  AL(delta, S * e->Hq);
  AL(dq, S * e->q_dim);
  AL(dh1, S * h);
  AL(rope_tab, (size_t)e->max_pos * (e->d / 2));
  AL(tp_sync, 64);
  AL(ipc_flags, 64);
  AL(tp_stage, e->tp_size > 1 ? (std::max(T, S) + 8) * h : 1);
  // dS^T tiles: [kv heads][64-row query tiles of a window][keys (L_max rounded to 128)][64]
  AL(d_meta, e->meta_bytes);
  if (measure) *total = pl.used;
#undef AL
}

size_t meta_size(const cs_engine* e) {
  const size_t T = e->T_max, S = e->max_seg;
  size_t b = 0;
  b += T * 4 * 4;                          // tokens, row_pos, row_seg, row_slot
  b += S * sizeof(cs::AttnSeg);
  b += (size_t)e->npages * 4 + 4096 * 4;   // page table (upper bound)
  b += 65536 * sizeof(cs::AttnWork) + 16384 * sizeof(cs::AttnDecWork);
  b += 8192 * sizeof(cs::AttnCombine);
  b += S * 4 * 2;                          // samp idx
  b += (size_t)e->L_max * 4;               // targets
  return (b + 4095) & ~size_t(4095);
}

}  // namespace

// =============================================================================== create
namespace {
using CommFactory = std::function<cs::Comm*(std::string*)>;

int create_engine(const cs_model_config* cfg, int device, int tp_rank, int tp_size,
                  const CommFactory& make_comm, cs_engine** out) {
  if (!cfg || !out) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: null argument");
  const cs_model_config& c = *cfg;
  if (c.n_layers < 1 || c.hidden < 1 || c.n_heads < 1 || c.n_kv_heads < 1 || c.head_dim < 1 ||
      c.ffn < 1 || c.vocab < 1)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: dimensions must be >= 1");
  if (c.lora_rank < 1 || c.lora_rank > 16)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: lora_rank must be in [1, 16]");
  if (c.n_heads % c.n_kv_heads != 0)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: kv heads must divide heads");
  if (c.head_dim != 64 && c.head_dim != 128)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: head_dim must be 64 or 128");
  if (c.n_heads / c.n_kv_heads > 64)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: GQA group too large");
  if (c.hidden > 8192)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: hidden must be <= 8192");
  if ((c.hidden % 64) != 0 || (c.ffn % 64) != 0 || (c.vocab % 8) != 0)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT,
                         "cs_engine_create: hidden/ffn must be multiples of 64, vocab of 8");
  if (c.page_size < 1 || c.n_pages < 1 || c.max_tokens < 1 || c.max_ft_len < 1)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: bad pool / capacity sizes");
  if (tp_size < 1 || tp_size > 8 || tp_rank < 0 || tp_rank >= tp_size)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create: need 0 <= tp_rank < tp_size <= 8");
  if (c.n_kv_heads % tp_size != 0 || c.ffn % tp_size != 0 || ((c.ffn / tp_size) % 64) != 0)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT,
                         "cs_engine_create: tp_size must divide the kv heads and ffn/tp_size be a multiple of 64");
  cs_engine* e = new cs_engine();
  e->cfg = c;
  e->device = device;
  e->tp_rank = tp_rank;
  e->tp_size = tp_size;
  e->Hq_g = c.n_heads;
  e->Hkv_g = c.n_kv_heads;
  e->f_g = c.ffn;
  e->h = c.hidden;
  e->Hq = c.n_heads / tp_size;
  e->Hkv = c.n_kv_heads / tp_size;
  e->d = c.head_dim;
  e->q_dim = e->Hq * c.head_dim;
  e->kv_dim = e->Hkv * c.head_dim;
  e->nqkv = e->q_dim + 2 * e->kv_dim;
  e->f = c.ffn / tp_size;
  e->V = c.vocab;
  e->r = c.lora_rank;
  e->NL = c.n_layers;
  e->P = c.page_size;
  e->npages = c.n_pages;
  e->swiglu = c.act == 1;
  e->norm = c.norm == 1;
  e->rope = c.rope == 1;
  e->gu_n = e->swiglu ? 2 * e->f : e->f;
  e->f_cat = e->f + 64;
  e->h_cat = e->h + 64;
  e->grp = e->Hq / e->Hkv;
  e->T_max = c.max_tokens;
  e->L_max = c.max_ft_len;
  e->S_max = std::max(c.max_tokens, 64);
  e->max_seg = std::max(c.max_segments, 1);
  e->head_chunk = std::min(1024, std::max(64, c.max_tokens));
  e->max_pos = std::max((long)c.max_ft_len, std::min<long>((long)c.n_pages * c.page_size, 1 << 17)) + 1;
  e->meta_bytes = meta_size(e);
  if (const char* v = std::getenv("CS_ATTN_TC")) e->use_tc_attn = std::atoi(v) != 0;
  if (const char* v = std::getenv("CS_ATTN_DEC")) e->use_dec_attn = std::atoi(v) != 0;
  e->down_rows = e->h + 64;

  if (cudaSetDevice(device) != cudaSuccess) {
    delete e;
    return cs::set_error(CS_ERR_CUDA, "cs_engine_create: cudaSetDevice failed");
  }
  if (tp_size > 1) {
    std::string err;
    e->comm = make_comm(&err);
    if (!e->comm) {
      delete e;
      return cs::set_error(CS_ERR_NCCL, "cs_engine_create: " + err);
    }
    // CS_TP_FUSED=0 keeps GEMM + separate all-reduce on peer-memory groups (A/B)
    const char* v = std::getenv("CS_TP_FUSED");
    e->tp_fused_allowed = !(v && std::atoi(v) == 0);
    e->tp_fused = e->comm->peer_capable() && e->tp_fused_allowed;  // IPC groups: after attach
  }
  size_t total = 0;
  layout(e, true, &total);
  e->arena_bytes = total;
  cudaError_t err = cudaMalloc(&e->arena, total);
  if (err != cudaSuccess) {
    delete e->comm;
    delete e;
    return cs::set_error(CS_ERR_OOM, "cs_engine_create: cudaMalloc(" + std::to_string(total) +
                                         ") failed: " + cudaGetErrorString(err));
  }
  layout(e, false, nullptr);
  if (e->comm) e->comm->bind_arena(e->arena, e->arena_bytes, e->ipc_flags);
  cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&e->st2, cudaStreamNonBlocking);
  cudaEventCreate(&e->ev0);
  cudaEventCreate(&e->ev1);
  cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming);
  cudaMallocHost(&e->h_meta, e->meta_bytes);
  cudaMallocHost(&e->h_loss, (size_t)e->L_max * sizeof(float));
  // zero everything that has padding semantics (concat pad columns, LoRA state, norms)
  cudaMemsetAsync(e->arena, 0, e->arena_used, e->st);
  // RoPE table in double precision on the host
  {
    const int half = e->d / 2;
    std::vector<float2> tab((size_t)e->max_pos * half);
    for (int p = 0; p < e->max_pos; ++p)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow((double)c.rope_theta, -(2.0 * i) / (double)e->d);
        const double ang = (double)p * inv;
        tab[(size_t)p * half + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
    cudaMemcpyAsync(e->rope_tab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice,
                    e->st);
    cudaStreamSynchronize(e->st);
  }
  cs::fill_f32(e->g1, (long)e->NL * e->h, 1.f, e->st);
  cs::fill_f32(e->g2, (long)e->NL * e->h, 1.f, e->st);
  cs::fill_f32(e->gf, e->h, 1.f, e->st);
  err = cudaStreamSynchronize(e->st);
  if (err != cudaSuccess) {
    cudaFree(e->arena);
    delete e->comm;
    delete e;
    return cs::set_error(CS_ERR_CUDA, std::string("cs_engine_create: ") + cudaGetErrorString(err));
  }
  *out = e;
  return CS_OK;
}
}  // namespace

struct cs_tp_group {
  cs::LocalGroup* g;
};

extern "C" int cs_engine_create(const cs_model_config* cfg, int device, int tp_rank, int tp_size,
                                const void* nccl_unique_id, cs_engine** out) {
  if (tp_size > 1 && !nccl_unique_id)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT,
                         "cs_engine_create: tp_size > 1 needs the NCCL unique id (or cs_engine_create_tp_local)");
  return create_engine(cfg, device, tp_rank, tp_size,
                       [&](std::string* err) { return cs::make_nccl_comm(nccl_unique_id, tp_rank, tp_size, err); },
                       out);
}

extern "C" int cs_nccl_unique_id(void* out128) {
  if (!out128) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_nccl_unique_id: null buffer");
  std::string err;
  if (cs::nccl_unique_id(out128, &err) != 0) return cs::set_error(CS_ERR_NCCL, err);
  return CS_OK;
}

extern "C" int cs_tp_group_create(int tp_size, cs_tp_group** out) {
  if (!out) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_tp_group_create: null argument");
  std::string err;
  cs::LocalGroup* g = cs::local_group_create(tp_size, &err);
  if (!g) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_tp_group_create: " + err);
  *out = new cs_tp_group{g};
  return CS_OK;
}

extern "C" int cs_tp_group_destroy(cs_tp_group* g) {
  if (!g) return CS_OK;
  cs::local_group_destroy(g->g);
  delete g;
  return CS_OK;
}

extern "C" int cs_engine_create_tp_local(const cs_model_config* cfg, int device, int tp_rank,
                                         cs_tp_group* group, cs_engine** out) {
  if (!group) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_engine_create_tp_local: null group");
  const int n = cs::local_group_size(group->g);
  return create_engine(cfg, device, tp_rank, n,
                       [&](std::string* err) { return cs::make_local_comm(group->g, tp_rank, device, err); },
                       out);
}

extern "C" int cs_engine_create_ipc(const cs_model_config* cfg, int device, int tp_rank, int tp_size,
                                    cs_engine** out) {
  return create_engine(cfg, device, tp_rank, tp_size,
                       [&](std::string* err) { return cs::make_ipc_comm(tp_rank, tp_size, device, err); },
                       out);
}

extern "C" int cs_engine_ipc_handle(cs_engine* e, void* out64, int64_t* arena_bytes) {
  if (!e || !out64 || !arena_bytes) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "ipc_handle: null argument");
  if (!e->comm) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "ipc_handle: not a tensor-parallel engine");
  CS_CUDA_TRY(cudaSetDevice(e->device));
  std::string err;
  if (e->comm->ipc_handle(out64, &err) != 0) return cs::set_error(CS_ERR_INVALID_ARGUMENT, err);
  *arena_bytes = (int64_t)e->arena_bytes;
  return CS_OK;
}

extern "C" int cs_engine_ipc_attach(cs_engine* e, const void* handles, const int64_t* arena_bytes) {
  if (!e || !handles || !arena_bytes) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "ipc_attach: null argument");
  if (!e->comm) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "ipc_attach: not a tensor-parallel engine");
  CS_CUDA_TRY(cudaSetDevice(e->device));
  std::string err;
  if (e->comm->ipc_attach(handles, arena_bytes, &err) != 0) return cs::set_error(CS_ERR_RUNTIME, err);
  e->tp_fused = e->comm->peer_capable() && e->tp_fused_allowed;
  return CS_OK;
}

extern "C" int cs_engine_set_profiling(cs_engine* e, int on) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "set_profiling: null engine");
  cudaStreamSynchronize(e->st);
  prof_collect(e);
  e->profiling = on != 0;
  for (int k = 0; k < cs_engine::kKinds; ++k)
    e->prof_ms[k] = e->prof_flops[k] = e->prof_bytes[k] = 0, e->prof_n[k] = 0;
  return CS_OK;
}

extern "C" int cs_engine_read_profile(cs_engine* e, int kind, double* ms, double* flops,
                                      double* bytes, int64_t* launches) {
  if (!e || kind < 0 || kind >= cs_engine::kKinds) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "read_profile: bad kind");
  if (ms) *ms = e->prof_ms[kind];
  if (flops) *flops = e->prof_flops[kind];
  if (bytes) *bytes = e->prof_bytes[kind];
  if (launches) *launches = e->prof_n[kind];
  return CS_OK;
}

// Matrix::alloc_hook (matrix.hpp:16-25): report every device buffer the engine owns.  All of
// them are carved from one arena at create time, so a cs_step / backward window allocates
// nothing; the audit lets tests prove no frozen-weight gradient buffer exists (graph pruning).
extern "C" int cs_engine_alloc_audit(cs_engine* e, cs_alloc_hook hook, void* user,
                                     int64_t* transient_allocs) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "alloc_audit: null engine");
  if (hook)
    for (const auto& a : e->audit) hook(a.name, a.elems, a.elem_bytes, user);
  if (transient_allocs) *transient_allocs = e->transient_allocs;
  return CS_OK;
}

extern "C" int64_t cs_engine_launch_count(cs_engine* e) {
  (void)e;
  return cs::g_launches.load();
}

extern "C" int cs_engine_pool_info(cs_engine* e, int32_t* n_layers, int32_t* vocab,
                                   int32_t* page_size, int64_t* n_pages) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "pool_info: null engine");
  if (n_layers) *n_layers = e->NL;
  if (vocab) *vocab = e->V;
  if (page_size) *page_size = e->P;
  if (n_pages) *n_pages = e->npages;
  return CS_OK;
}

// Max over the TP group of n <= 8 host doubles (identical result on every rank; no-op at
// tp_size 1).  The co-serving loop of a TP group runs once per rank and must plan the same
// iteration on every rank: its clock (step wall / device ms) is made rank-invariant here.
// Sum-only all-reduce: each rank writes its values into its own slot of a zeroed
// [ranks][8] buffer, the sum then holds every rank's values, the host takes the max.
extern "C" int cs_engine_tp_sync_max(cs_engine* e, double* vals, int n) {
  if (!e || (!vals && n > 0) || n < 0 || n > 8)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "tp_sync_max: need an engine and 0 <= n <= 8");
  if (!e->comm || n == 0) return CS_OK;
  CS_CUDA_TRY(cudaSetDevice(e->device));
  float h[64] = {};
  for (int i = 0; i < n; ++i) h[e->tp_rank * 8 + i] = (float)vals[i];
  CS_CUDA_TRY(cudaMemcpyAsync(e->tp_sync, h, sizeof(h), cudaMemcpyHostToDevice, e->st));
  std::string err;
  if (e->comm->allreduce_f32(e->tp_sync, 8 * e->tp_size, e->st, &err) != 0)
    return cs::set_error(CS_ERR_NCCL, "tp_sync_max: " + err);
  CS_CUDA_TRY(cudaMemcpyAsync(h, e->tp_sync, sizeof(h), cudaMemcpyDeviceToHost, e->st));
  CS_CUDA_TRY(cudaStreamSynchronize(e->st));
  for (int i = 0; i < n; ++i) {
    float m = h[i];
    for (int rk = 1; rk < e->tp_size; ++rk) m = std::max(m, h[rk * 8 + i]);
    vals[i] = (double)m;
  }
  return CS_OK;
}

extern "C" int cs_engine_destroy(cs_engine* e) {
  if (!e) return CS_OK;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->st);
  cudaFree(e->arena);
  cudaFreeHost(e->h_meta);
  cudaFreeHost(e->h_loss);
  cudaEventDestroy(e->ev0);
  cudaEventDestroy(e->ev1);
  cudaEventDestroy(e->ev_fork);
  cudaEventDestroy(e->ev_join);
  cudaStreamDestroy(e->st2);
  cudaStreamDestroy(e->st);
  delete e->comm;
  delete e;
  return CS_OK;
}

// =============================================================================== weights
namespace {
int refresh_lora(cs_engine* e, int update, float lr, float b1, float b2, float eps) {
  cs::AdamParams p;
  p.A = e->loraA;
  p.B = e->loraB;
  p.gA = e->gA;
  p.gB = e->gB;
  p.mA = e->mA;
  p.vA = e->vA;
  p.mB = e->mB;
  p.vB = e->vB;
  p.A_t = e->A_t;
  p.B_t = e->B_t;
  p.down_cat = e->down_cat;
  p.down_rows = e->down_rows;
  p.n_layers = e->NL;
  p.f = e->f;
  p.r = e->r;
  p.h = e->h;
  p.lr = lr;
  p.b1 = b1;
  p.b2 = b2;
  p.eps = eps;
  p.bc1 = update ? 1.f - std::pow(b1, (float)e->adam_t) : 1.f;
  p.bc2 = update ? 1.f - std::pow(b2, (float)e->adam_t) : 1.f;
  cs::adam_step(p, update, e->st);
  CS_CUDA_TRY(cudaGetLastError());
  return CS_OK;
}
}  // namespace

extern "C" int cs_engine_set_weight(cs_engine* e, const char* name, int layer, const void* host,
                                    int dtype, int64_t rows, int64_t cols) {
  if (!e || !name || !host) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "set_weight: null argument");
  if (dtype != 0 && dtype != 1) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "set_weight: dtype must be 0 (f64) or 1 (f32)");
  const std::string n(name);
  const bool global = (n == "embed" || n == "unembed" || n == "final_norm");
  if (!global && (layer < 0 || layer >= e->NL))
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "set_weight: layer out of range");
  const long count = rows * cols;
  // whole-model shapes (reference layout [in, out]); TP ranks keep their shard below
  const long h = e->h, V = e->V, r = e->r, d = e->d;
  const long qd_g = (long)e->Hq_g * d, kvd_g = (long)e->Hkv_g * d, f_g = e->f_g;
  auto expect = [&](long er, long ec) -> bool { return rows == er && cols == ec; };
  auto bad = [&]() {
    return cs::set_error(CS_ERR_INVALID_ARGUMENT,
                         "set_weight: unexpected shape for '" + n + "' [" + std::to_string(rows) +
                             "," + std::to_string(cols) + "]");
  };
  // shard: rows [r0, r0+nr) x cols [c0, c0+nc) of the whole matrix (vectors: cols)
  const long rk = e->tp_rank;
  long r0 = 0, nr = rows, c0 = 0, nc = cols;
  if (n == "embed") {
    if (!expect(V, h)) return bad();
  } else if (n == "unembed") {
    if (!expect(h, V)) return bad();
  } else if (n == "final_norm" || n == "norm1" || n == "norm2") {
    if (count != h) return bad();
    nr = 1, nc = h;
  } else if (n == "wq") {
    if (!expect(h, qd_g)) return bad();
    c0 = rk * e->q_dim, nc = e->q_dim;
  } else if (n == "wk" || n == "wv") {
    if (!expect(h, kvd_g)) return bad();
    c0 = rk * e->kv_dim, nc = e->kv_dim;
  } else if (n == "bq") {
    if (count != qd_g) return bad();
    nr = 1, c0 = rk * e->q_dim, nc = e->q_dim;
  } else if (n == "bk" || n == "bv") {
    if (count != kvd_g) return bad();
    nr = 1, c0 = rk * e->kv_dim, nc = e->kv_dim;
  } else if (n == "wo") {
    if (!expect(qd_g, h)) return bad();
    r0 = rk * e->q_dim, nr = e->q_dim;
  } else if (n == "w_gate" || n == "w_up") {
    if (n == "w_gate" && !e->swiglu)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "set_weight: w_gate given for a ReLU model");
    if (!expect(h, f_g)) return bad();
    c0 = rk * e->f, nc = e->f;
  } else if (n == "w_down") {
    if (!expect(f_g, h)) return bad();
    r0 = rk * e->f, nr = e->f;
  } else if (n == "lora_a") {
    if (!expect(f_g, r)) return bad();
    r0 = rk * e->f, nr = e->f;
  } else if (n == "lora_b") {
    if (!expect(r, h)) return bad();
  } else {
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "set_weight: unknown weight '" + n + "'");
  }
  const long src_cols = (nr == 1 && rows != 1 && cols == 1) ? rows : cols;  // column vectors
  std::vector<float> f32((size_t)nr * nc);
  for (long i = 0; i < nr; ++i)
    for (long j = 0; j < nc; ++j) {
      const long k = (r0 + i) * src_cols + (c0 + j);
      f32[(size_t)i * nc + j] = dtype == 0 ? (float)static_cast<const double*>(host)[k]
                                           : static_cast<const float*>(host)[k];
    }
  const long lr = nr, lc = nc, lcount = nr * nc;
  const int L = layer;
  const long qd = e->q_dim, kvd = e->kv_dim, f = e->f;
  float* stage = nullptr;
  CS_CUDA_TRY(cudaSetDevice(e->device));
  CS_CUDA_TRY(cudaMalloc(&stage, lcount * sizeof(float)));
  e->transient_allocs += 1;
  // stream-ordered upload: the engine stream is non-blocking w.r.t. the legacy stream
  CS_CUDA_TRY(cudaMemcpyAsync(stage, f32.data(), lcount * sizeof(float), cudaMemcpyHostToDevice,
                              e->st));
  int rc = CS_OK;
  cudaStream_t st = e->st;
  if (n == "embed") {
    cs::cast_f32_bf16(stage, lr, lc, e->embed, h, 0, st);
  } else if (n == "unembed") {
    cs::cast_f32_bf16(stage, lr, lc, e->unembed_t, h, 1, st);
  } else if (n == "final_norm") {
    cudaMemcpyAsync(e->gf, stage, h * 4, cudaMemcpyDeviceToDevice, st);
  } else if (n == "wq" || n == "wk" || n == "wv") {
    const long off = n == "wq" ? 0 : (n == "wk" ? qd : qd + kvd);
    cs::cast_f32_bf16(stage, lr, lc, e->wqkv_t + ((size_t)L * e->nqkv + off) * h, h, 1, st);
  } else if (n == "wo") {
    cs::cast_f32_bf16(stage, lr, lc, e->wo_t + (size_t)L * h * qd, qd, 1, st);
  } else if (n == "w_gate" || n == "w_up") {
    if (e->swiglu)  // interleaved 64-row blocks [gate | up] (kernels.h EPI_SWIGLU)
      cs::cast_f32_bf16_interleaved(stage, lr, lc, e->wgu_t + (size_t)L * e->gu_n * h, h, 128,
                                    n == "w_up" ? 64 : 0, st);
    else
      cs::cast_f32_bf16(stage, lr, lc, e->wgu_t + (size_t)L * e->gu_n * h, h, 1, st);
  } else if (n == "w_down") {
    cs::cast_f32_bf16(stage, lr, lc, e->down_cat + (size_t)L * e->down_rows * e->f_cat, e->f_cat, 1, st);
  } else if (n == "lora_a") {
    cudaMemcpyAsync(e->loraA + (size_t)L * f * r, stage, lcount * 4, cudaMemcpyDeviceToDevice, st);
    rc = refresh_lora(e, 0, 0, 0, 0, 0);
  } else if (n == "lora_b") {
    cudaMemcpyAsync(e->loraB + (size_t)L * r * h, stage, lcount * 4, cudaMemcpyDeviceToDevice, st);
    rc = refresh_lora(e, 0, 0, 0, 0, 0);
  } else if (n == "bq" || n == "bk" || n == "bv") {
    const long off = n == "bq" ? 0 : (n == "bk" ? qd : qd + kvd);
    cudaMemcpyAsync(e->bqkv + (size_t)L * e->nqkv + off, stage, lcount * 4, cudaMemcpyDeviceToDevice, st);
  } else if (n == "norm1" || n == "norm2") {
    cudaMemcpyAsync((n == "norm1" ? e->g1 : e->g2) + (size_t)L * h, stage, h * 4,
                    cudaMemcpyDeviceToDevice, st);
  }
  cudaStreamSynchronize(st);
  cudaFree(stage);
  CS_CUDA_TRY(cudaGetLastError());
  return rc;
}

extern "C" int cs_engine_init_random(cs_engine* e, uint64_t seed) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "init_random: null engine");
  cudaStream_t st = e->st;
  const float ws = 1.f / std::sqrt((float)e->h);
  const float wf = 1.f / std::sqrt((float)e->f_g);
  const size_t NL = e->NL;
  CS_CUDA_TRY(cudaSetDevice(e->device));
  // TP: sharded matrices draw per-rank streams; replicated ones (embed, unembed, B) share one
  const uint64_t ss = seed + 7919ull * (uint64_t)e->tp_rank;
  // tiny_model.hpp:51-63 scales; the forward/backward layouts hold identical values
  cs::init_normal_bf16(e->embed, (long)e->V * e->h, ws, seed + 1, st);
  cs::init_normal_bf16(e->unembed_t, (long)e->V * e->h, ws, seed + 2, st);
  cs::init_normal_bf16(e->wqkv_t, (long)(NL * e->nqkv * e->h), ws, ss + 3, st);
  cs::init_normal_bf16(e->wo_t, (long)(NL * e->q_dim * e->h), ws, ss + 4, st);
  cs::init_normal_bf16(e->wgu_t, (long)(NL * e->gu_n * e->h), ws, ss + 5, st);
  // down: fill whole concat buffers, then the LoRA columns are rewritten by refresh_lora;
  // pad columns [f + r, f + 64) must stay zero -> fill per row via cast of random fp32
  {
    float* tmp = nullptr;
    CS_CUDA_TRY(cudaMalloc(&tmp, (size_t)e->f * e->h * sizeof(float)));
    e->transient_allocs += 1;
    for (size_t l = 0; l < NL; ++l) {
      cs::init_normal_f32(tmp, (long)e->f * e->h, wf, ss + 100 + l, st);
      cs::cast_f32_bf16(tmp, e->f, e->h, e->down_cat + l * e->down_rows * e->f_cat, e->f_cat, 1, st);
    }
    cudaStreamSynchronize(st);
    cudaFree(tmp);
  }
  cs::init_normal_f32(e->loraA, (long)(NL * e->f * e->r), 0.2f * wf, ss + 6, st);
  cs::init_normal_f32(e->loraB, (long)(NL * e->r * e->h), 0.2f, seed + 7, st);
  if (e->cfg.qkv_bias) cs::init_normal_f32(e->bqkv, (long)(NL * e->nqkv), 0.02f, ss + 8, st);
  int rc = refresh_lora(e, 0, 0, 0, 0, 0);
  if (rc) return rc;
  CS_CUDA_TRY(cudaStreamSynchronize(st));
  return CS_OK;
}

extern "C" int cs_engine_get_lora(cs_engine* e, int layer, double* a_out, double* b_out) {
  if (!e || layer < 0 || layer >= e->NL)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "get_lora: bad engine/layer");
  cudaStreamSynchronize(e->st);
  const size_t na = (size_t)e->f * e->r, nb = (size_t)e->r * e->h;
  std::vector<float> t(std::max(na, nb));
  if (a_out) {
    CS_CUDA_TRY(cudaMemcpy(t.data(), e->loraA + layer * na, na * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < na; ++i) a_out[i] = t[i];
  }
  if (b_out) {
    CS_CUDA_TRY(cudaMemcpy(t.data(), e->loraB + layer * nb, nb * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nb; ++i) b_out[i] = t[i];
  }
  return CS_OK;
}

// =============================================================================== step
namespace {

struct StepPlan {
  int T = 0;
  int n_seg = 0;
  int ft_row0 = 0;  // first FT forward row (== T if none)
  int ad_row0 = 0;  // first adapter row (== T if none)
  int n_samp = 0;
  int n_work = 0, n_comb = 0, n_tc = 0, n_dec = 0, n_comb_tc = 0;
  // device pointers into d_meta
  int *tokens, *row_pos, *row_seg, *row_slot, *page_table, *samp_idx, *targets;
  cs::AttnSeg* segs;
  cs::AttnWork* work;
  cs::AttnWork* work_tc;
  cs::AttnDecWork* work_dec;
  int dec_max_rows = 0;
  int comb_slices = 4;  // 16-row slices of the largest decode / legacy combine item
  cs::AttnCombine* comb;
  cs::AttnCombine* comb_tc;  // split-KV parts of the tcgen05 kernel (256-row parts)
  std::vector<int> samp_seg;  // segment of each sampled row
};

int gemm(cs_engine* e, const void* A, long lda, long a_rows, const void* B, long ldb, long b_rows,
         void* C, long ldc, long M, long N, long K, int epi, const float* bias = nullptr,
         const cs::GemmScatter* sc = nullptr, int b_mn = 0, void* C2 = nullptr, long ldc2 = 0,
         int c2_row0 = 0, const cs::QkvEpi* qkv = nullptr) {
  cs::GemmDesc g;
  if (sc) g.scatter = *sc;
  g.b_mn = b_mn;
  g.A = A;
  g.lda = lda;
  g.a_rows = a_rows;
  g.B = B;
  g.ldb = ldb;
  g.b_rows = b_rows;
  g.C = C;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.epi = epi;
  g.bias = bias;
  g.b_const = 1;  // every engine GEMM's B operand is a (frozen or LoRA) weight
  if (qkv) g.qkv = *qkv;
  if (epi == cs::EPI_SWIGLU) {  // m = silu(gate) * up into C, the FT rows' gate / up into C2
    g.C2 = C2;
    g.ldc2 = ldc2;
    g.c2_row0 = c2_row0;
    g.m_cols = (int)(N / 2);
  }
  e->launches++;
  cs_engine::ProfRec pr{};
  if (e->profiling) {
    pr.flops = 2.0 * (double)M * (double)N * (double)K;
    pr.bytes = 2.0 * ((double)M * K + (double)N * K) +
               (double)M * N * (epi == cs::EPI_SWIGLU ? 1 : epi == cs::EPI_BF16 ? 2 : 4);
    pr.kind = 0;
    pr.m = M, pr.n = N, pr.k = K, pr.epi = (int)epi;
    prof_begin(e, pr);
  }
  cudaError_t err = cs::gemm_tn(g, e->st);
  if (e->profiling) prof_end(e, pr);
  if (err != cudaSuccess)
    return cs::set_error(CS_ERR_CUDA, std::string("gemm: ") + cudaGetErrorString(err));
  return CS_OK;
}

#define TRY(x)            \
  do {                    \
    int _rc = (x);        \
    if (_rc) return _rc;  \
  } while (0)

// in-place sum of buf[0, n) over the TP ranks (no-op at tp_size 1); SURVEY.md §8e
int tp_allreduce(cs_engine* e, float* buf, size_t n) {
  if (!e->comm || n == 0) return CS_OK;
  cs_engine::ProfRec pr{};
  if (e->profiling) {
    pr.bytes = 2.0 * (double)n * 4.0 * (e->tp_size - 1) / e->tp_size;  // ring bus bytes
    pr.kind = 4;
    prof_begin(e, pr);
  }
  std::string err;
  const int rc = e->comm->allreduce_f32(buf, n, e->st, &err);
  if (e->profiling) prof_end(e, pr);
  if (rc != 0) return cs::set_error(CS_ERR_NCCL, "tp all-reduce: " + err);
  return CS_OK;
}

// row-parallel projections add into the replicated residual stream: rank 0 accumulates
// (x += p_0), the other ranks overwrite (x = p_r); the all-reduce then leaves x + sum_r p_r
int rowpar_epi(const cs_engine* e) { return (e->comm && e->tp_rank != 0) ? cs::EPI_F32 : cs::EPI_F32_ADD; }

// Row-parallel GEMM whose fp32 output is summed over the TP ranks into dst [M, h] (add_old:
// dst += sum_r partial_r, the replicated residual stream; else dst = sum_r partial_r).
// Peer-memory groups run it FUSED: the GEMM epilogue stores each
// partial tile straight into the owning rank's staging slot over NVLink (rows are owned in
// M / ranks blocks) while the other tiles are still in the tensor pipe; after a cross-rank
// stream barrier each owner sums its rows' slots in rank order and stores the result into
// every rank's dst (peer stores), then a second barrier.  Otherwise (NCCL, tp 1, or
// CS_TP_FUSED=0): GEMM into dst + in-place all-reduce.
int tp_rowpar(cs_engine* e, const void* A, long lda, long a_rows, const void* B, long ldb,
              long b_rows, float* dst, long M, long K, bool add_old, int b_mn = 0) {
  const long h = e->h;
  if (!e->tp_fused) {
    const int epi = add_old ? rowpar_epi(e) : cs::EPI_F32;
    TRY(gemm(e, A, lda, a_rows, B, ldb, b_rows, dst, h, M, h, K, epi, nullptr, nullptr, b_mn));
    return tp_allreduce(e, dst, (size_t)M * h);
  }
  if (M <= 0) return CS_OK;
  std::string err;
  const int n = e->tp_size;
  if (!e->stage_tab[0]) {
    void* out[8] = {};
    if (e->comm->exchange_ptr(e->tp_stage, out, &err) != 0) return cs::set_error(CS_ERR_NCCL, err);
    for (int j = 0; j < n; ++j) e->stage_tab[j] = static_cast<float*>(out[j]);
  }
  const std::vector<float*>* dtab = nullptr;
  for (const auto& d : e->dst_tabs)
    if (d.first == dst) dtab = &d.second;
  if (!dtab) {
    void* out[8] = {};
    if (e->comm->exchange_ptr(dst, out, &err) != 0) return cs::set_error(CS_ERR_NCCL, err);
    std::vector<float*> t(n);
    for (int j = 0; j < n; ++j) t[j] = static_cast<float*>(out[j]);
    e->dst_tabs.emplace_back(dst, std::move(t));
    dtab = &e->dst_tabs.back().second;
  }
  const int rpo = (int)((M + n - 1) / n);
  cs::GemmScatter sc;
  for (int j = 0; j < n; ++j) sc.peer[j] = e->stage_tab[j];
  sc.rows_per_owner = rpo;
  sc.rank = e->tp_rank;
  cs_engine::ProfRec pr{};
  TRY(gemm(e, A, lda, a_rows, B, ldb, b_rows, nullptr, h, M, h, K, cs::EPI_F32_SCATTER, nullptr, &sc, b_mn));
  if (e->profiling) {
    pr.bytes = 2.0 * (double)M * h * 4.0 * (n - 1) / n;
    pr.kind = 4;
    prof_begin(e, pr);
  }
  if (e->comm->stream_barrier(e->st, &err) != 0) return cs::set_error(CS_ERR_NCCL, err);
  CS_CUDA_TRY(cs::tp_reduce_bcast(e->tp_stage, h, n, e->tp_rank, rpo, (int)M, (int)h, dtab->data(), h,
                                  add_old ? 1 : 0, e->st));
  if (e->comm->stream_barrier(e->st, &err) != 0) return cs::set_error(CS_ERR_NCCL, err);
  if (e->profiling) prof_end(e, pr);
  return CS_OK;
}

int prepare(cs_engine* e, const cs_iteration_plan* plan, StepPlan& sp) {
  const int T = plan->n_tokens;
  if (T < 0 || T > e->T_max)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: n_tokens out of range [0, max_tokens]");
  if (plan->n_segments < 0 || plan->n_segments > e->max_seg)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: too many segments");
  if (T > 0 && (!plan->tokens || !plan->segments))
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: null tokens/segments");
  sp.T = T;
  sp.n_seg = plan->n_segments;
  sp.ft_row0 = T;
  sp.ad_row0 = T;
  const int P = e->P;
  const int ptl = plan->page_table_len;
  if (ptl < 0 || ptl > e->npages + 4096)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: page_table_len out of range");
  // host staging layout
  uint8_t* hb = e->h_meta;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return o;
  };
  const size_t o_tok = take((size_t)T * 4), o_pos = take((size_t)T * 4), o_seg = take((size_t)T * 4);
  const size_t o_slot = take((size_t)T * 4);  // KV-pool row of each token (QKV epilogue append)
  const size_t o_segs = take((size_t)sp.n_seg * sizeof(cs::AttnSeg));
  const size_t o_pt = take((size_t)ptl * 4);
  int* h_tok = reinterpret_cast<int*>(hb + o_tok);
  int* h_pos = reinterpret_cast<int*>(hb + o_pos);
  int* h_rseg = reinterpret_cast<int*>(hb + o_seg);
  int* h_slot = reinterpret_cast<int*>(hb + o_slot);
  cs::AttnSeg* h_segs = reinterpret_cast<cs::AttnSeg*>(hb + o_segs);
  if (ptl) std::memcpy(hb + o_pt, plan->page_table, (size_t)ptl * 4);
  for (int i = 0; i < ptl; ++i)
    if (plan->page_table[i] < 0 || plan->page_table[i] >= e->npages)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: page id out of range");
  int row = 0;
  bool in_adapter_suffix = false;
  std::vector<int> samp_rows;
  std::vector<cs::AttnWork> work, work_tc, work_dec;
  std::vector<cs::AttnCombine> comb, comb_tc;
  const int rpt = 64 / e->grp;
  // tcgen05 attention items: two 128-row query tiles per CTA share every K/V tile (one tile per
  // CTA for small calls measured slightly negative in the bench); the key-range split below
  // spreads small calls over the SMs
  const int rpt_tc = 2 * (128 / e->grp);
  const bool tc_ok = e->d == 128 && (e->P % 16) == 0 && e->use_tc_attn;
  double attn_flops = 0, attn_bytes = 0, tc_flops = 0, tc_bytes = 0;
  for (int s = 0; s < sp.n_seg; ++s) {
    const cs_segment& g = plan->segments[s];
    if (g.q_start != row || g.q_len < 1 || g.q_start + g.q_len > T)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT,
                           "cs_step: segments must tile the token batch contiguously in order");
    if (g.kind < CS_SEG_DECODE || g.kind > CS_SEG_FT_FWD)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: bad segment kind");
    if (g.kind == CS_SEG_DECODE && g.q_len != 1)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: decode segment with q_len != 1");
    const long need = g.ctx_start + g.q_len;
    if (g.ctx_start < 0 || g.page_off < 0 || g.n_pages < 0 || g.page_off + g.n_pages > ptl ||
        (long)g.n_pages * P < need)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: segment page table does not cover its context");
    if (need >= e->max_pos)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: context longer than the RoPE table");
    if (g.adapter) in_adapter_suffix = true;
    else if (in_adapter_suffix)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: adapter segments must form a suffix of the batch");
    if (g.adapter && sp.ad_row0 == T) sp.ad_row0 = g.q_start;
    if (g.kind == CS_SEG_FT_FWD) {
      if (s != sp.n_seg - 1)
        return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: the FT forward segment must be last");
      if (!g.adapter)
        return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: FT rows must use the adapter");
      sp.ft_row0 = g.q_start;
    }
    h_segs[s] = cs::AttnSeg{g.q_start, g.q_len, g.ctx_start, g.page_off};
    for (int i = 0; i < g.q_len; ++i) {
      const int t = plan->tokens[row + i];
      if (t < 0 || t >= e->V) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: token id out of range");
      h_tok[row + i] = t;
      h_pos[row + i] = g.ctx_start + i;
      h_rseg[row + i] = s;
      const int pos = g.ctx_start + i;
      h_slot[row + i] = plan->page_table[g.page_off + pos / P] * P + pos % P;
    }
    if (g.sample) {
      samp_rows.push_back(row + g.q_len - 1);
      sp.samp_seg.push_back(s);
    }
    {  // algorithmic attention work of this segment per layer
      const double ql = g.q_len, c0 = g.ctx_start;
      const double fl = 4.0 * e->Hq * e->d * (ql * c0 + ql * (ql + 1) / 2.0);
      const double by = (c0 + ql) * (double)e->kv_dim * 2.0 * 2.0 + ql * e->q_dim * 2.0 * 2.0;
      if (tc_ok && g.q_len >= 16) {
        tc_flops += fl;
        tc_bytes += by;
      } else {
        attn_flops += fl;
        attn_bytes += by;
      }
    }
    // attention work items (GQA-packed q tiles x kv heads): multi-row segments on the
    // tcgen05 kernel (128 packed rows), decode rows on the bandwidth kernel (64 packed rows)
    if (tc_ok && g.q_len >= 16) {
      for (int q0 = 0; q0 < g.q_len; q0 += rpt_tc) {
        const int nq = std::min(rpt_tc, g.q_len - q0);
        const int nkeys = g.ctx_start + q0 + nq;
        for (int kh = 0; kh < e->Hkv; ++kh)
          work_tc.push_back(cs::AttnWork{s, q0, nq, kh, 0, nkeys, -1, 0});
      }
    } else if (g.q_len * e->grp <= 16 && e->use_dec_attn && (P % 16) == 0) {
      // decode kernel: the whole GQA-packed segment fits one m16 tile
      for (int kh = 0; kh < e->Hkv; ++kh)
        work_dec.push_back(cs::AttnWork{s, 0, g.q_len, kh, 0, g.ctx_start + g.q_len, -1, 0});
    } else {
      for (int q0 = 0; q0 < g.q_len; q0 += rpt) {
        const int nq = std::min(rpt, g.q_len - q0);
        const int nkeys = g.ctx_start + q0 + nq;
        for (int kh = 0; kh < e->Hkv; ++kh)
          work.push_back(cs::AttnWork{s, q0, nq, kh, 0, nkeys, -1, 0});
      }
    }
    row += g.q_len;
  }
  if (row != T) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: segments do not cover n_tokens");
  e->step_attn_flops = attn_flops;
  e->step_attn_bytes = attn_bytes;
  e->step_tc_flops = tc_flops;
  e->step_tc_bytes = tc_bytes;
  // split long key ranges when the grid is small (flash-decoding)
  {
    const int target = 2 * 148;
    const int n0 = (int)work.size();
    if (n0 > 0 && n0 < target) {
      const int factor = (target + n0 - 1) / n0;
      std::vector<cs::AttnWork> w2;
      int part = 0;
      for (const auto& w : work) {
        const int tiles = (w.k_end + 63) / 64;
        const int ns = std::min(factor, std::max(1, tiles / 4));
        if (ns <= 1) {
          w2.push_back(w);
          continue;
        }
        const int per = (tiles + ns - 1) / ns;
        int p0 = part;
        int cnt = 0;
        for (int t = 0; t < tiles; t += per) {
          cs::AttnWork x = w;
          x.k_begin = t * 64;
          x.k_end = std::min(w.k_end, (t + per) * 64);
          x.part = part++;
          w2.push_back(x);
          ++cnt;
        }
        comb.push_back(cs::AttnCombine{w.seg, w.q0, w.nq, w.kv_head, p0, cnt, 0, 0});
      }
      if (part <= 4096) work.swap(w2);
      else comb.clear();
    }
  }
  // decode: balance the 32-key tiles over the SMs -- split long key ranges into parts of
  // `chunk` keys (multiples of 128 = one tile per warp) so that the grid is ~8 waves of
  // 1 CTA/SM (small wave-quantisation tail, longest parts first), but no part is shorter
  // than 512 keys (4 tiles per warp: the per-warp TMA ring stays full)
  {
    int dec_kt = 32, dec_nw = 4, dec_cps = 1, dec_stream = 0;
    cs::attn_decode_geometry(e->d, &dec_kt, &dec_nw, &dec_cps, &dec_stream);
    long total = 0;
    for (const auto& w : work_dec) total += w.k_end;
    // per-item CTAs: ~8 waves of CTAs; persistent streams (one warp per item): ~2 parts per
    // warp of the grid (scripts/decode_variants.py A/B over CS_DEC_TARGET 1/2/3/6: 2 is the
    // best compromise between balance and combine work)
    static const long stream_mult = [] {  // CS_DEC_TARGET: items per warp of the stream grid
      const char* v = std::getenv("CS_DEC_TARGET");
      return v ? std::max(1L, std::atol(v)) : 2L;
    }();
    const long target = dec_stream ? stream_mult * 148 * dec_cps * dec_nw : 8L * 148 * dec_cps;
    const long tile_round = dec_stream ? (long)dec_kt : (long)dec_kt * dec_nw;
    long chunk = (total + target - 1) / target;
    chunk = std::max<long>(4 * tile_round, (chunk + tile_round - 1) / tile_round * tile_round);
    int part = 0;
    for (const auto& c : comb) part = std::max(part, c.part0 + c.n_parts);
    std::vector<cs::AttnWork> w2;
    w2.reserve(work_dec.size());
    for (const auto& w : work_dec) {
      // balanced parts (multiples of 128 keys), none a sliver: round(k_end / chunk)
      const int ns = (int)std::max<long>(1, (w.k_end + chunk / 2) / chunk);
      if (ns <= 1 || part + ns > 4096) {
        w2.push_back(w);
        continue;
      }
      const long per = ((w.k_end + ns - 1) / ns + tile_round - 1) / tile_round * tile_round;
      const int p0 = part;
      for (int t = 0; t < ns && t * per < w.k_end; ++t) {
        cs::AttnWork x = w;
        x.k_begin = (int)(t * per);
        x.k_end = (int)std::min<long>(w.k_end, (t + 1) * per);
        x.part = part++;
        w2.push_back(x);
      }
      comb.push_back(cs::AttnCombine{w.seg, w.q0, w.nq, w.kv_head, p0, part - p0, 0, 0});
    }
    // longest first: the heaviest CTAs start in the first wave
    std::stable_sort(w2.begin(), w2.end(), [](const cs::AttnWork& x, const cs::AttnWork& y) {
      return x.k_end - x.k_begin > y.k_end - y.k_begin;
    });
    if (dec_stream) {
      // the stream warps take items w, w + W, w + 2W, ... (W = warps of the grid): reverse every
      // second round of W so each warp pairs a long item with a short one (boustrophedon):
      // 1-1.5% per launch at the bench's operating point (profiles/r2_decode_timeline.txt)
      const long n = (long)w2.size();
      const long grid = std::min<long>((n + dec_nw - 1) / dec_nw, 148L * dec_cps);
      const long W = grid * dec_nw;
      for (long r0 = W; r0 < n; r0 += 2 * W) std::reverse(w2.begin() + r0, w2.begin() + std::min(n, r0 + W));
    }
    work_dec.swap(w2);
  }
  // tcgen05 items: split key ranges (flash-decoding style; parts merged by the LSE combine) by
  // a makespan model of the launch: a part of t 128-key tiles costs t + kFix tile-times (TMEM /
  // barrier setup, the two Q tiles, first K/V latency, epilogue), parts go to the 148 SMs
  // longest first (the block scheduler's greedy order = LPT), a split adds the combine launch
  // (kComb) and each split part its fp32 partial round trip (kPer).  Constants fitted on 48
  // launches of scripts/attn_mix_bench.py (8B, windows 512-2048 at context 0-7680, with and
  // without a prefill chunk; 2.3% mean error): 1 tile = 2.6 us, kFix 4.5, kComb 4.3, kPer 0.01.
  // Candidates: no split, and parts capped at T / (148 m) tiles or at the longest item / k.
  // (The earlier fixed rules -- >= 1024-key parts over ~2 waves below 148 items, halves to fill
  // the last wave below 444 -- split a 1024-token window at 4K context into 1.7 waves of
  // halves: 145 us vs 121 us unsplit.)
  if (!work_tc.empty()) {
    constexpr double kFix = 4.5, kComb = 4.3, kPer = 0.01;
    constexpr int kSMs = 148;
    std::vector<int> t(work_tc.size());
    long T = 0;
    int tmax = 0;
    for (size_t i = 0; i < work_tc.size(); ++i) {
      t[i] = (work_tc[i].k_end - work_tc[i].k_begin + 127) / 128;
      T += t[i];
      tmax = std::max(tmax, t[i]);
    }
    std::vector<double> cost, load(kSMs);
    auto makespan = [&](int cap, int* n_parts) {
      cost.clear();
      int n_split = 0;
      for (int x : t) {
        const int ns = (x + cap - 1) / cap, per = (x + ns - 1) / ns;
        if (ns > 1) n_split += ns;
        for (int k = 0, left = x; k < ns; ++k, left -= per) cost.push_back(std::min(per, left) + kFix);
      }
      *n_parts = (int)cost.size();
      std::sort(cost.begin(), cost.end(), std::greater<double>());
      // greedy onto the least-loaded SM (min-heap of loads)
      std::fill(load.begin(), load.end(), 0.0);
      double mx = 0.0;
      for (double c : cost) {
        std::pop_heap(load.begin(), load.end(), std::greater<double>());
        load.back() += c;
        mx = std::max(mx, load.back());
        std::push_heap(load.begin(), load.end(), std::greater<double>());
      }
      return mx + (n_split ? kComb + kPer * n_split : 0.0);
    };
    int best_cap = tmax, best_parts = 0;
    double best = makespan(tmax, &best_parts);
    std::vector<int> caps;
    for (int m : {1, 2, 3, 4, 6, 8}) caps.push_back((int)((T + (long)kSMs * m - 1) / ((long)kSMs * m)));
    for (int k : {2, 3, 4}) caps.push_back((tmax + k - 1) / k);
    for (int cap : caps) {
      if (cap < 2 || cap >= tmax) continue;
      int np = 0;
      const double ms = makespan(cap, &np);
      if (np <= 1024 && ms < best - 1e-9) best = ms, best_cap = cap, best_parts = np;
    }
    if (best_cap < tmax) {
      int part = 0;
      std::vector<cs::AttnWork> w2;
      for (size_t i = 0; i < work_tc.size(); ++i) {
        const cs::AttnWork& w = work_tc[i];
        const int ns = (t[i] + best_cap - 1) / best_cap;
        if (ns <= 1) {
          w2.push_back(w);
          continue;
        }
        const int per = (t[i] + ns - 1) / ns;
        const int p0 = part;
        for (int k = 0; k < ns; ++k) {
          cs::AttnWork x = w;
          x.k_begin = w.k_begin + k * per * 128;
          x.k_end = std::min(w.k_end, w.k_begin + (k + 1) * per * 128);
          if (x.k_begin >= x.k_end) break;
          x.part = part++;
          w2.push_back(x);
        }
        comb_tc.push_back(cs::AttnCombine{w.seg, w.q0, w.nq, w.kv_head, p0, part - p0, 0, 0});
      }
      work_tc.swap(w2);
    }
  }
  // longest key ranges first (causal tiles have very different lengths)
  std::stable_sort(work_tc.begin(), work_tc.end(),
                   [](const cs::AttnWork& x, const cs::AttnWork& y) {
                     return x.k_end - x.k_begin > y.k_end - y.k_begin;
                   });
  sp.n_work = (int)work.size();
  sp.n_tc = (int)work_tc.size();
  sp.n_dec = (int)work_dec.size();
  sp.dec_max_rows = 0;
  for (const auto& w : work_dec) sp.dec_max_rows = std::max(sp.dec_max_rows, w.nq * e->grp);
  {
    int mr = 1;
    for (const auto& c : comb) mr = std::max(mr, c.nq * e->grp);
    sp.comb_slices = (mr + 15) / 16;
  }
  sp.n_comb = (int)comb.size();
  sp.n_comb_tc = (int)comb_tc.size();
  if (sp.n_work + sp.n_tc + sp.n_dec > 65536 || sp.n_comb + sp.n_comb_tc > 8192)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: attention work list too large");
  const size_t o_work = take(work.size() * sizeof(cs::AttnWork));
  const size_t o_wtc = take(work_tc.size() * sizeof(cs::AttnWork));
  const size_t o_wdec = take(work_dec.size() * sizeof(cs::AttnDecWork));
  const size_t o_comb = take(comb.size() * sizeof(cs::AttnCombine));
  const size_t o_comb_tc = take(comb_tc.size() * sizeof(cs::AttnCombine));
  const size_t o_samp = take(samp_rows.size() * 4);
  const int ft_s = (plan->ft.phase == CS_FT_FORWARD) ? plan->ft.s : 0;
  const size_t o_tg = take((size_t)std::max(ft_s, 0) * 4);
  if (off > e->meta_bytes) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: plan too large");
  if (!work.empty()) std::memcpy(hb + o_work, work.data(), work.size() * sizeof(cs::AttnWork));
  if (!work_tc.empty()) std::memcpy(hb + o_wtc, work_tc.data(), work_tc.size() * sizeof(cs::AttnWork));
  if (!work_dec.empty()) {  // resolve segment fields and the first boxes' pool rows (P % 16 == 0)
    cs::AttnDecWork* dw = reinterpret_cast<cs::AttnDecWork*>(hb + o_wdec);
    for (size_t i = 0; i < work_dec.size(); ++i) {
      const cs::AttnWork& w = work_dec[i];
      const cs::AttnSeg& g = h_segs[w.seg];
      cs::AttnDecWork d{};
      d.q_row = g.q_start + w.q0;
      d.pos0 = g.ctx_start + w.q0;
      d.page_off = g.page_off;
      d.kv_head = w.kv_head;
      d.k_begin = w.k_begin;
      d.k_end = w.k_end;
      d.part = w.part;
      d.nq = w.nq;
      const int last_box = (w.k_end - 1) & ~15;
      for (int b = 0; b < 8; ++b) {
        const int jb = std::min(w.k_begin + 16 * b, last_box);
        d.prow[b] = plan->page_table[g.page_off + jb / P] * P + jb % P;
      }
      dw[i] = d;
    }
  }
  if (!comb_tc.empty()) std::memcpy(hb + o_comb_tc, comb_tc.data(), comb_tc.size() * sizeof(cs::AttnCombine));
  if (!comb.empty()) std::memcpy(hb + o_comb, comb.data(), comb.size() * sizeof(cs::AttnCombine));
  if (!samp_rows.empty()) std::memcpy(hb + o_samp, samp_rows.data(), samp_rows.size() * 4);
  if (ft_s > 0) {
    if (!plan->ft.targets) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: FT forward window without targets");
    for (int i = 0; i < ft_s; ++i) {
      const int t = plan->ft.targets[i];
      if (t >= e->V) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: target id out of range");
    }
    std::memcpy(hb + o_tg, plan->ft.targets, (size_t)ft_s * 4);
  }
  sp.n_samp = (int)samp_rows.size();
  cudaError_t err = cudaMemcpyAsync(e->d_meta, hb, off, cudaMemcpyHostToDevice, e->st);
  if (err != cudaSuccess) return cs::set_error(CS_ERR_CUDA, "cs_step: meta upload failed");
  uint8_t* db = e->d_meta;
  sp.tokens = reinterpret_cast<int*>(db + o_tok);
  sp.row_pos = reinterpret_cast<int*>(db + o_pos);
  sp.row_seg = reinterpret_cast<int*>(db + o_seg);
  sp.row_slot = reinterpret_cast<int*>(db + o_slot);
  sp.segs = reinterpret_cast<cs::AttnSeg*>(db + o_segs);
  sp.page_table = reinterpret_cast<int*>(db + o_pt);
  sp.work = reinterpret_cast<cs::AttnWork*>(db + o_work);
  sp.comb = reinterpret_cast<cs::AttnCombine*>(db + o_comb);
  sp.comb_tc = reinterpret_cast<cs::AttnCombine*>(db + o_comb_tc);
  sp.work_tc = reinterpret_cast<cs::AttnWork*>(db + o_wtc);
  sp.work_dec = reinterpret_cast<cs::AttnDecWork*>(db + o_wdec);
  sp.samp_idx = reinterpret_cast<int*>(db + o_samp);
  sp.targets = reinterpret_cast<int*>(db + o_tg);
  return CS_OK;
}

// copy `rows` contiguous rows of width `w` elements (row stride ld_src) into dst rows
template <typename T>
void save_rows(cs_engine* e, T* dst, long ld_dst, const T* src, long ld_src, int rows, long w) {
  if (rows <= 0) return;
  cudaMemcpy2DAsync(dst, ld_dst * sizeof(T), src, ld_src * sizeof(T), w * sizeof(T), rows,
                    cudaMemcpyDeviceToDevice, e->st);
}

int forward(cs_engine* e, const cs_iteration_plan* plan, StepPlan& sp, double* loss_sum) {
  const int T = sp.T;
  const long h = e->h, f = e->f, r = e->r;
  const int n_ft = T - sp.ft_row0;
  const int n_ad = T - sp.ad_row0;
  const int l0 = plan->ft.l;  // FT window start position
  cudaStream_t st = e->st;
  cs::embed_gather(sp.tokens, e->embed, e->x, T, h, st);
  const float eps = e->cfg.rms_eps;
  const size_t kv_layer = (size_t)e->npages * e->P * e->kv_dim;
  for (int l = 0; l < e->NL; ++l) {
    const bool keep_attn = l > 0;  // pruning: layer 0 needs no attention backward
    // ---- attention block
    cs::rmsnorm_cast(e->x, h, e->g1 + (size_t)l * h, e->xb, h, e->rstd, T, h, eps, e->norm, st);
    if (n_ft > 0 && keep_attn) {
      if (e->norm) {
        save_rows(e, e->ft_x + ((size_t)l * e->L_max + l0) * h, h, e->x + (size_t)sp.ft_row0 * h, h, n_ft, h);
        save_rows(e, e->ft_rstd1 + (size_t)l * e->L_max + l0, 1, e->rstd + sp.ft_row0, 1, n_ft, 1);
      }
    }
    cs::RopeAppendParams rp;
    rp.qkv = e->qkv;
    rp.ld = e->nqkv;
    rp.row_pos = sp.row_pos;
    rp.row_seg = sp.row_seg;
    rp.segs = sp.segs;
    rp.page_table = sp.page_table;
    rp.k_pool = e->k_pool + l * kv_layer;
    rp.v_pool = e->v_pool + l * kv_layer;
    rp.page_size = e->P;
    rp.n_heads = e->Hq;
    rp.n_kv_heads = e->Hkv;
    rp.head_dim = e->d;
    rp.use_rope = e->rope;
    rp.rope_theta = e->cfg.rope_theta;
    rp.T = T;
    rp.ft_row0 = sp.ft_row0;
    rp.q_cache = (n_ft > 0 && keep_attn) ? e->ft_q + (size_t)l * e->L_max * e->q_dim : nullptr;
    const float* qkv_bias = e->cfg.qkv_bias ? e->bqkv + (size_t)l * e->nqkv : nullptr;
    if (e->d == 128) {
      // RoPE and the KV append in the QKV GEMM's epilogue (kernels.h EPI_QKV_ROPE)
      cs::QkvEpi qe;
      qe.row_pos = rp.row_pos;
      qe.row_slot = sp.row_slot;
      qe.k_pool = rp.k_pool;
      qe.v_pool = rp.v_pool;
      qe.q_cache = rp.q_cache;
      qe.rope_tab = e->rope_tab;
      qe.q_dim = e->q_dim;
      qe.kv_dim = e->kv_dim;
      qe.ft_row0 = sp.ft_row0;
      qe.use_rope = e->rope;
      TRY(gemm(e, e->xb, h, e->T_max, e->wqkv_t + (size_t)l * e->nqkv * h, h, e->nqkv, e->qkv, e->nqkv,
               T, e->nqkv, h, cs::EPI_QKV_ROPE, qkv_bias, nullptr, 0, nullptr, 0, 0, &qe));
    } else {
      TRY(gemm(e, e->xb, h, e->T_max, e->wqkv_t + (size_t)l * e->nqkv * h, h, e->nqkv, e->qkv, e->nqkv,
               T, e->nqkv, h, cs::EPI_BF16, qkv_bias));
      cs::rope_append(rp, st);
    }
    cs::AttnFwdParams ap;
    ap.q = e->qkv;
    ap.q_ld = e->nqkv;
    ap.k_pool = rp.k_pool;
    ap.v_pool = rp.v_pool;
    ap.kv_dim = e->kv_dim;
    ap.page_size = e->P;
    ap.page_table = sp.page_table;
    ap.segs = sp.segs;
    ap.work = sp.work;
    ap.combine = sp.comb;
    ap.out = e->attn;
    ap.out_ld = e->q_dim;
    ap.lse = e->lse;
    ap.lse_ld = e->Hq;
    ap.part_o = e->part_o;
    ap.part_lse = e->part_lse;
    ap.grp = e->grp;
    ap.comb_slices = sp.comb_slices;
    ap.scale_log2 = (float)(1.0 / std::sqrt((double)e->d) * 1.4426950408889634);
    cs_engine::ProfRec apr{};
    const bool bw_attn = sp.n_work + sp.n_dec > 0;
    // spatial sharing inside the step: the HBM-bound decode (and small-segment) attention runs
    // on a side stream next to the tensor-bound FT-window attention, on the SMs the latter's
    // grid leaves free (profiling runs keep one stream: its events serialise anyway)
    const bool fork = bw_attn && sp.n_tc > 0 && !e->profiling;
    cudaStream_t sa = fork ? e->st2 : st;
    if (fork) {
      CS_CUDA_TRY(cudaEventRecord(e->ev_fork, st));
      CS_CUDA_TRY(cudaStreamWaitEvent(e->st2, e->ev_fork, 0));
    }
    if (e->profiling && bw_attn) {
      apr.flops = e->step_attn_flops;
      apr.bytes = e->step_attn_bytes;
      apr.kind = 1;
      prof_begin(e, apr);
    }
    if (sp.n_dec > 0) {
      cs::AttnFwdParams dp = ap;
      dp.dwork = sp.work_dec;
      dp.max_dec_rows = sp.dec_max_rows;
      CUtensorMap mk, mv;
      const long pool_rows = (long)e->npages * e->P;
      if (cs::make_map(&mk, rp.k_pool, pool_rows, e->kv_dim, e->kv_dim, 16) != 0 ||
          cs::make_map(&mv, rp.v_pool, pool_rows, e->kv_dim, e->kv_dim, 16) != 0)
        return cs::set_error(CS_ERR_CUDA, "decode attention: TMA map creation failed");
      cs_engine::ProfRec dpr{};
      if (e->profiling) {
        dpr.bytes = e->step_attn_bytes;  // decode rows' K/V bytes (the bandwidth kernel's share)
        dpr.flops = e->step_attn_flops;
        dpr.kind = 5;
        prof_begin(e, dpr);
      }
      CS_CUDA_TRY(cs::attn_decode(dp, mk, mv, e->d, sp.n_dec, sa));
      if (e->profiling) prof_end(e, dpr);
    }
    CS_CUDA_TRY(cs::attn_fwd(ap, e->d, sp.n_work, sp.n_comb, sa));
    if (e->profiling && bw_attn) prof_end(e, apr);
    if (fork) CS_CUDA_TRY(cudaEventRecord(e->ev_join, sa));
    if (sp.n_tc > 0) {
      CUtensorMap mk, mv, mk128, mv128;
      const long pool_rows = (long)e->npages * e->P;
      if (cs::make_map(&mk, rp.k_pool, pool_rows, e->kv_dim, e->kv_dim, 16) != 0 ||
          cs::make_map(&mv, rp.v_pool, pool_rows, e->kv_dim, e->kv_dim, 16) != 0 ||
          cs::make_map(&mk128, rp.k_pool, pool_rows, e->kv_dim, e->kv_dim, 128) != 0 ||
          cs::make_map(&mv128, rp.v_pool, pool_rows, e->kv_dim, e->kv_dim, 128) != 0)
        return cs::set_error(CS_ERR_CUDA, "attention: TMA map creation failed");
      cs::AttnFwdParams tp = ap;
      tp.work = sp.work_tc;
      tp.part_o = e->part_o_tc;
      tp.part_lse = e->part_lse_tc;
      cs_engine::ProfRec tpr{};
      if (e->profiling) {
        tpr.flops = e->step_tc_flops;
        tpr.bytes = e->step_tc_bytes;
        tpr.kind = 3;
        prof_begin(e, tpr);
      }
      CS_CUDA_TRY(cs::attn_fwd_tc2(tp, mk, mv, mk128, mv128, sp.n_tc, st));
      if (sp.n_comb_tc > 0) {
        cs::AttnFwdParams cp = tp;
        cp.combine = sp.comb_tc;
        cp.part_rows = 256;
        CS_CUDA_TRY(cs::attn_combine(cp, e->d, sp.n_comb_tc, st));
      }
      if (e->profiling) prof_end(e, tpr);
    }
    if (fork) CS_CUDA_TRY(cudaStreamWaitEvent(st, e->ev_join, 0));
    if (n_ft > 0 && keep_attn) {
      save_rows(e, e->ft_o + ((size_t)l * e->L_max + l0) * e->q_dim, e->q_dim,
                e->attn + (size_t)sp.ft_row0 * e->q_dim, e->q_dim, n_ft, e->q_dim);
      save_rows(e, e->ft_lse + ((size_t)l * e->L_max + l0) * e->Hq, e->Hq,
                e->lse + (size_t)sp.ft_row0 * e->Hq, e->Hq, n_ft, e->Hq);
    }
    TRY(tp_rowpar(e, e->attn, e->q_dim, e->T_max, e->wo_t + (size_t)l * h * e->q_dim, e->q_dim, h, e->x,
                  T, e->q_dim, true));
    // ---- MLP block
    if (n_ft > 0 && e->norm)
      save_rows(e, e->ft_r1 + ((size_t)l * e->L_max + l0) * h, h, e->x + (size_t)sp.ft_row0 * h, h, n_ft, h);
    cs::rmsnorm_cast(e->x, h, e->g2 + (size_t)l * h, e->xb, h, e->rstd, T, h, eps, e->norm, st);
    if (n_ft > 0 && e->norm)
      save_rows(e, e->ft_rstd2 + (size_t)l * e->L_max + l0, 1, e->rstd + sp.ft_row0, 1, n_ft, 1);
    if (e->swiglu) {
      // gate||up with the SwiGLU in the epilogue: m straight from the accumulators (pad
      // columns zeroed), the FT rows' bf16 gate / up saved for the backward (tiny_model.hpp:205)
      TRY(gemm(e, e->xb, h, e->T_max, e->wgu_t + (size_t)l * e->gu_n * h, h, e->gu_n, e->m, e->f_cat,
               T, e->gu_n, h, cs::EPI_SWIGLU, nullptr, nullptr, 0,
               n_ft > 0 ? e->ft_gu + ((size_t)l * e->L_max + l0) * e->gu_n : nullptr, e->gu_n,
               n_ft > 0 ? sp.ft_row0 : T));
    } else {
      TRY(gemm(e, e->xb, h, e->T_max, e->wgu_t + (size_t)l * e->gu_n * h, h, e->gu_n, e->gu, e->gu_n,
               T, e->gu_n, h, cs::EPI_BF16));
      if (n_ft > 0)
        save_rows(e, e->ft_gu + ((size_t)l * e->L_max + l0) * e->gu_n, e->gu_n,
                  e->gu + (size_t)sp.ft_row0 * e->gu_n, e->gu_n, n_ft, e->gu_n);
      cs::act_fwd(e->gu, e->gu_n, e->m, e->f_cat, T, f, e->swiglu, st);
    }
    if (n_ad > 0) {
      // u = m A for adapter rows (segmented LoRA down, tiny_model.hpp:207)
      TRY(gemm(e, e->m + (size_t)sp.ad_row0 * e->f_cat, e->f_cat, e->T_max - sp.ad_row0,
               e->A_t + (size_t)l * 16 * f, f, r, e->lu, r, n_ad, r, f, cs::EPI_F32));
      cs::lora_pack(e->lu, r, e->m + (size_t)sp.ad_row0 * e->f_cat, e->f_cat, f, n_ad, st);
      if (n_ft > 0)
        save_rows(e, e->ft_lu + ((size_t)l * e->L_max + l0) * r, r,
                  e->lu + (size_t)(sp.ft_row0 - sp.ad_row0) * r, r, n_ft, r);
    }
    // x += [m | u] [W_down ; B] (tiny_model.hpp:206-211 as one K-concatenated GEMM)
    TRY(tp_rowpar(e, e->m, e->f_cat, e->T_max, e->down_cat + (size_t)l * e->down_rows * e->f_cat, e->f_cat, h,
                  e->x, T, e->f_cat, true));
  }
  // ---- sampled rows: final norm -> logits -> argmax
  if (sp.n_samp > 0) {
    cs::rmsnorm_cast_gather(e->x, h, sp.samp_idx, e->gf, e->hf, h, nullptr, sp.n_samp, h, eps,
                            e->norm, st);
    TRY(gemm(e, e->hf, h, std::max(e->head_chunk, e->max_seg), e->unembed_t, h, e->V,
             e->samp_logits, e->V, sp.n_samp, e->V, h, cs::EPI_F32));
    cs::argmax_rows(e->samp_logits, e->V, sp.n_samp, e->V, e->next_tok, e->amax_part, st);
  }
  // ---- FT rows: fused generative loss + loss-head gradient into dY (top layer)
  if (n_ft > 0) {
    const int L = plan->ft.seq_len;
    const float inv = L > 1 ? 1.f / (float)(L - 1) : 0.f;
    for (int c0 = 0; c0 < n_ft; c0 += e->head_chunk) {
      const int cn = std::min(e->head_chunk, n_ft - c0);
      const float* xs = e->x + (size_t)(sp.ft_row0 + c0) * h;
      cs::rmsnorm_cast(xs, h, e->gf, e->hf, h, e->hrstd, cn, h, eps, e->norm, st);
      TRY(gemm(e, e->hf, h, std::max(e->head_chunk, e->max_seg), e->unembed_t, h, e->V, e->logits,
               e->V, cn, e->V, h, cs::EPI_F32));
      cs::ce_fwd_bwd(e->logits, e->V, sp.targets + c0, cn, e->V, inv, e->loss_rows + c0, e->dlog,
                     e->V, st);
      // dH = dlogits . U^T, U^T read from the [V, h] forward copy (MN-major)
      TRY(gemm(e, e->dlog, e->V, e->head_chunk, e->unembed_t, h, e->V, e->dh, h, cn, h, e->V,
               cs::EPI_F32, nullptr, nullptr, 1));
      cs::rms_bwd_add(nullptr, 0, xs, h, e->gf, e->hrstd, e->dh, h,
                      e->dy[e->dy_cur] + (size_t)(l0 + c0) * h, h, nullptr, 0, cn, h, e->norm, st);
    }
    e->h_loss_n = n_ft;
    CS_CUDA_TRY(cudaMemcpyAsync(e->h_loss, e->loss_rows, n_ft * 4, cudaMemcpyDeviceToHost, st));
  }
  (void)loss_sum;
  return CS_OK;
}

int backward_window(cs_engine* e, const cs_iteration_plan* plan, StepPlan& sp) {
  const cs_ft_window& w = plan->ft;
  const int n = w.layer, b = w.l, s = w.s, a = b - s;
  cudaStream_t st = e->st;
  const long h = e->h, f = e->f, r = e->r;
  const int L = e->ft_L;
  // ---- dependency / ordering checks
  if (e->bwd_layer == -2) {
    if (e->ft_len != L || L <= 0)
      return cs::set_error(CS_ERR_ORDERING, "backward window before the forward pass completed");
    e->bwd_layer = e->NL - 1;
    e->bwd_next_end = L;
  }
  if (e->bwd_layer < 0) return cs::set_error(CS_ERR_ORDERING, "backward already complete; run cs_adam_step");
  if (n != e->bwd_layer || b != e->bwd_next_end || s < 1 || a < 0)
    return cs::set_error(CS_ERR_ORDERING,
                         "backward window out of order: expected layer " + std::to_string(e->bwd_layer) +
                             " ending at " + std::to_string(e->bwd_next_end));
  if (s > e->S_max) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "backward window larger than max_tokens");
  if (w.page_off < 0 || w.n_pages < 0 || w.page_off + w.n_pages > plan->page_table_len ||
      (long)w.n_pages * e->P < L)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "backward window: FT page table does not cover L");
  if (b == L) {  // first window of this layer: fresh ΔKVAccum
    CS_CUDA_TRY(cudaMemsetAsync(e->dk_acc, 0, (size_t)L * e->kv_dim * 4, st));
    CS_CUDA_TRY(cudaMemsetAsync(e->dv_acc, 0, (size_t)L * e->kv_dim * 4, st));
  }
  const float* Y = e->dy[e->dy_cur] + (size_t)a * h;  // dLoss/d(out of layer n), rows [a,b)
  float* Xout = e->dy[e->dy_cur ^ 1] + (size_t)a * h;
  const size_t Lm = e->L_max;
  // ---- MLP + LoRA (tiny_model.hpp:276-287)
  // dycat = [bf16(dY) | bf16(dY B^T)] (tiny_model.hpp:281): dlu on the tensor cores (N = r),
  // dB += u^T dY (:280) on the CUDA cores
  cs::lora_db(Y, h, e->ft_lu + ((size_t)n * Lm + a) * r, r, s, h, e->gB + (size_t)n * r * h,
              e->dycat, e->h_cat, st);
  TRY(gemm(e, e->dycat, e->h_cat, e->S_max, e->B_t + (size_t)n * 16 * h, h, 16, e->dlu, r, s, r, h,
           cs::EPI_F32));
  cs::lora_pack(e->dlu, r, e->dycat, e->h_cat, h, s, st);
  // dm = [dY | dU] . [W_down^T ; A^T]: down_cat's [h + 64, f] block, MN-major
  TRY(gemm(e, e->dycat, e->h_cat, e->S_max, e->down_cat + (size_t)n * e->down_rows * e->f_cat,
           e->f_cat, e->h_cat, e->dm, f, s, f, e->h_cat, cs::EPI_BF16, nullptr, nullptr, 1));
  cs::mlp_bwd(e->dm, f, e->ft_gu + ((size_t)n * Lm + a) * e->gu_n, e->gu_n, e->dlu, r, e->dgu,
              e->gu_n, e->gA + (size_t)n * f * r, s, f, e->swiglu, st);
  if (n > 0) {
    TRY(tp_rowpar(e, e->dgu, e->gu_n, e->S_max, e->wgu_t + (size_t)n * e->gu_n * h, h, e->gu_n, e->dh2,
                  s, e->gu_n, false, 1));
    cs::rms_bwd_add(Y, h, e->ft_r1 + ((size_t)n * Lm + a) * h, h, e->g2 + (size_t)n * h,
                    e->ft_rstd2 + (size_t)n * Lm + a, e->dh2, h, e->dr1, h, e->dr1b, h, s, h,
                    e->norm, st);
    // ---- attention (tiny_model.hpp:289-315)
    TRY(gemm(e, e->dr1b, h, e->S_max, e->wo_t + (size_t)n * h * e->q_dim, e->q_dim, h, e->dO,
             e->q_dim, s, e->q_dim, h, cs::EPI_BF16, nullptr, nullptr, 1));
    const size_t kv_layer = (size_t)e->npages * e->P * e->kv_dim;
    cs::AttnBwdParams bp;
    bp.q_cache = e->ft_q + (size_t)n * Lm * e->q_dim;
    bp.q_ld = e->q_dim;
    bp.dO = e->dO;
    bp.do_ld = e->q_dim;
    bp.O = e->ft_o + ((size_t)n * Lm + a) * e->q_dim;
    bp.o_ld = e->q_dim;
    bp.lse = e->ft_lse + (size_t)n * Lm * e->Hq;
    bp.lse_ld = e->Hq;
    bp.delta = e->delta;
    bp.delta_ld = e->Hq;
    bp.k_pool = e->k_pool + n * kv_layer;
    bp.v_pool = e->v_pool + n * kv_layer;
    bp.kv_dim = e->kv_dim;
    bp.page_size = e->P;
    bp.page_table = sp.page_table;
    bp.page_off = w.page_off;
    bp.a = a;
    bp.b = b;
    bp.dq = e->dq;
    bp.dq_ld = e->q_dim;
    bp.dk_acc = e->dk_acc;
    bp.dv_acc = e->dv_acc;
    bp.acc_ld = e->kv_dim;
    bp.grp = e->grp;
    bp.scale = (float)(1.0 / std::sqrt((double)e->d));
    bp.scale_log2 = bp.scale * 1.4426950408889634f;
    cs_engine::ProfRec bpr{};
    if (e->profiling) {
      // algorithmic work (2.5x the forward): S = QK^T recompute, dP, dV, dK,
      // dQ -- 5 x 2*d per (q, k, head)
      const double pairs = (double)s * ((double)a + (s + 1) / 2.0);
      bpr.flops = 5.0 * 2.0 * e->d * e->Hq * pairs;
      bpr.bytes = 0;
      bpr.kind = 2;
      prof_begin(e, bpr);
    }
    // v2 takes any GQA group <= 8 (groups that do not divide 64 leave pad rows in a query
    // tile); the v1 kernels need 64 % group == 0
    const bool bwd_tc = e->use_tc_attn && e->d == 128 && (e->P % 16) == 0 && e->grp <= 8;
    if (bwd_tc) {
      CUtensorMap mk, mv, mk128, mv128, mq3, mo3;
      const long pool_rows = (long)e->npages * e->P;
      const int qbox = 64 / e->grp;  // 3-D boxes: 64 / grp positions x grp heads packed rows
      if (cs::make_map(&mk, bp.k_pool, pool_rows, e->kv_dim, e->kv_dim, 16) != 0 ||
          cs::make_map(&mv, bp.v_pool, pool_rows, e->kv_dim, e->kv_dim, 16) != 0 ||
          cs::make_map(&mk128, bp.k_pool, pool_rows, e->kv_dim, e->kv_dim, 128) != 0 ||
          cs::make_map(&mv128, bp.v_pool, pool_rows, e->kv_dim, e->kv_dim, 128) != 0 ||
          cs::make_map_3d(&mq3, bp.q_cache, 128, e->Hq, e->L_max, 256, (long)e->q_dim * 2, e->grp,
                          qbox) != 0 ||
          cs::make_map_3d(&mo3, bp.dO, 128, e->Hq, e->S_max, 256, (long)e->q_dim * 2, e->grp,
                          qbox) != 0)
        return cs::set_error(CS_ERR_CUDA, "attention backward: TMA map creation failed");
      CUtensorMap mdq;  // dK/dV/dQ in one kernel; dQ reduce-added into fp32
      if (cs::make_map_3d_f32(&mdq, bp.dq, e->d, e->Hq, s, (long)e->d * 4, bp.dq_ld * 4, 64, e->grp,
                              64 / e->grp) != 0)
        return cs::set_error(CS_ERR_CUDA, "attention backward: dQ TMA map creation failed");
      CS_CUDA_TRY(cs::attn_bwd_fused(bp, mk, mv, mk128, mv128, mq3, mo3, mdq, e->Hq, st));
    } else {
      CS_CUDA_TRY(cs::attn_bwd(bp, e->d, e->Hq, st));
    }
    if (e->profiling) prof_end(e, bpr);
    cs::rope_bwd_pack(e->dq, e->q_dim, e->dk_acc, e->dv_acc, e->kv_dim, a, s, e->Hq, e->Hkv, e->d,
                      e->rope, e->cfg.rope_theta, e->dqkv, e->nqkv, st);
    TRY(tp_rowpar(e, e->dqkv, e->nqkv, e->S_max, e->wqkv_t + (size_t)n * e->nqkv * h, h, e->nqkv,
                  e->dh1, s, e->nqkv, false, 1));
    cs::rms_bwd_add(e->dr1, h, e->ft_x + ((size_t)n * Lm + a) * h, h, e->g1 + (size_t)n * h,
                    e->ft_rstd1 + (size_t)n * Lm + a, e->dh1, h, Xout, h, nullptr, 0, s, h,
                    e->norm, st);
  }
  e->bwd_next_end = a;
  if (a == 0) {
    e->bwd_layer = n - 1;
    e->bwd_next_end = L;
    e->dy_cur ^= 1;
  }
  return CS_OK;
}

int step_impl(cs_engine* e, const cs_iteration_plan* plan, bool sync, cs_step_result* res) {
  if (!e || !plan) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: null argument");
  cudaSetDevice(e->device);
  cs::set_rope_table(e->rope_tab);
  const cs_ft_window& w = plan->ft;
  if (w.phase < CS_FT_NONE || w.phase > CS_FT_BACKWARD)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: bad FT phase");
  // FT forward bookkeeping (SPEC.md:283-291 cache-desync)
  if (w.phase == CS_FT_FORWARD) {
    if (w.seq_len < 1 || w.seq_len > e->L_max)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: FT seq_len out of range [1, max_ft_len]");
    if (e->bwd_layer != -2)
      return cs::set_error(CS_ERR_ORDERING, "cs_step: forward window while a backward pass is in flight");
    if (w.l == 0 && e->ft_len != 0 && e->ft_L != w.seq_len)
      return cs::set_error(CS_ERR_ORDERING, "cs_step: new mini-batch before the previous one finished");
    if (w.l != e->ft_len)
      return cs::set_error(CS_ERR_CACHE_DESYNC, "cs_step: cache length " + std::to_string(e->ft_len) +
                                                    " != l_i " + std::to_string(w.l));
    if (w.l + w.s > w.seq_len || w.s < 1)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: forward window exceeds seq_len");
    const cs_segment* last = plan->n_segments > 0 ? &plan->segments[plan->n_segments - 1] : nullptr;
    if (!last || last->kind != CS_SEG_FT_FWD || last->q_len != w.s || last->ctx_start != w.l)
      return cs::set_error(CS_ERR_INVALID_ARGUMENT,
                           "cs_step: FT forward window must be the last segment (q_len = s, ctx_start = l)");
  } else {
    for (int i = 0; i < plan->n_segments; ++i)
      if (plan->segments[i].kind == CS_SEG_FT_FWD)
        return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: FT segment without a forward window");
  }
  StepPlan sp;
  TRY(prepare(e, plan, sp));
  CS_CUDA_TRY(cudaEventRecord(e->ev0, e->st));
  if (w.phase == CS_FT_FORWARD && w.l == 0) {
    e->ft_L = w.seq_len;
    e->dy_cur = 0;
  }
  if (sp.T > 0) TRY(forward(e, plan, sp, nullptr));
  if (w.phase == CS_FT_FORWARD) e->ft_len = w.l + w.s;
  if (w.phase == CS_FT_BACKWARD) {
    TRY(backward_window(e, plan, sp));
    if (plan->n_extra_bwd < 0 || (plan->n_extra_bwd > 0 && !plan->extra_bwd))
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: bad extra backward windows");
    for (int i = 0; i < plan->n_extra_bwd; ++i) {
      cs_iteration_plan q = *plan;
      q.ft = plan->extra_bwd[i];
      q.ft.phase = CS_FT_BACKWARD;
      TRY(backward_window(e, &q, sp));
    }
  } else if (plan->n_extra_bwd > 0) {
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_step: extra backward windows without a backward phase");
  }
  CS_CUDA_TRY(cudaEventRecord(e->ev1, e->st));
  CS_CUDA_TRY(cudaGetLastError());
  if (!sync) return CS_OK;
  if (res) {
    if (res->next_tokens) {
      for (int s = 0; s < plan->n_segments; ++s) res->next_tokens[s] = -1;
      if (sp.n_samp > 0) {
        std::vector<int> nt(sp.n_samp);
        CS_CUDA_TRY(cudaMemcpyAsync(nt.data(), e->next_tok, sp.n_samp * 4, cudaMemcpyDeviceToHost, e->st));
        CS_CUDA_TRY(cudaStreamSynchronize(e->st));
        for (int i = 0; i < sp.n_samp; ++i) res->next_tokens[sp.samp_seg[i]] = nt[i];
      }
    }
    if (res->logits && sp.n_samp > 0)
      CS_CUDA_TRY(cudaMemcpyAsync(res->logits, e->samp_logits, (size_t)sp.n_samp * e->V * 4,
                                  cudaMemcpyDeviceToHost, e->st));
  }
  CS_CUDA_TRY(cudaStreamSynchronize(e->st));
  if (e->profiling) prof_collect(e);
  if (res) {
    double ls = 0.0;
    if (w.phase == CS_FT_FORWARD)
      for (int i = 0; i < std::min(e->h_loss_n, w.s); ++i) ls += e->h_loss[i];
    res->ft_loss_sum = ls;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e->ev0, e->ev1);
    res->iteration_ms = ms;
  }
  return CS_OK;
}

}  // namespace

extern "C" int cs_step(cs_engine* e, const cs_iteration_plan* plan, cs_step_result* result) {
  return step_impl(e, plan, true, result);
}

extern "C" int cs_step_async(cs_engine* e, const cs_iteration_plan* plan) {
  return step_impl(e, plan, false, nullptr);
}

extern "C" int cs_sync(cs_engine* e, cs_step_result* result) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_sync: null engine");
  CS_CUDA_TRY(cudaStreamSynchronize(e->st));
  if (e->profiling) prof_collect(e);
  if (result) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e->ev0, e->ev1);
    result->iteration_ms = ms;
  }
  return CS_OK;
}

extern "C" int cs_adam_step(cs_engine* e, float lr, float beta1, float beta2, float eps) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_adam_step: null engine");
  if (e->bwd_layer != -1)
    return cs::set_error(CS_ERR_ORDERING, "cs_adam_step: backward pass of the mini-batch not complete");
  CS_CUDA_TRY(cudaSetDevice(e->device));
  // TP: B is replicated and each rank holds the partial dB of its ffn shard (u = sum_r m_r A_r
  // folded into the down partial sums) -> one all-reduce per mini-batch; dA stays local
  TRY(tp_allreduce(e, e->gB, (size_t)e->NL * e->r * e->h));
  e->adam_t += 1;
  TRY(refresh_lora(e, 1, lr, beta1, beta2, eps));
  // mini-batch done: grads consumed, FT state reset
  CS_CUDA_TRY(cudaMemsetAsync(e->gA, 0, (size_t)e->NL * e->f * e->r * 4, e->st));
  CS_CUDA_TRY(cudaMemsetAsync(e->gB, 0, (size_t)e->NL * e->r * e->h * 4, e->st));
  e->ft_len = 0;
  e->ft_L = 0;
  e->bwd_layer = -2;
  e->bwd_next_end = 0;
  e->dy_cur = 0;
  CS_CUDA_TRY(cudaStreamSynchronize(e->st));
  return CS_OK;
}

extern "C" int cs_zero_lora_grads(cs_engine* e);
extern "C" int cs_engine_reset_ft(cs_engine* e) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "reset_ft: null engine");
  e->ft_len = 0;
  e->ft_L = 0;
  e->bwd_layer = -2;
  e->bwd_next_end = 0;
  e->dy_cur = 0;
  return cs_zero_lora_grads(e);
}

extern "C" int cs_zero_lora_grads(cs_engine* e) {
  if (!e) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "null engine");
  CS_CUDA_TRY(cudaMemsetAsync(e->gA, 0, (size_t)e->NL * e->f * e->r * 4, e->st));
  CS_CUDA_TRY(cudaMemsetAsync(e->gB, 0, (size_t)e->NL * e->r * e->h * 4, e->st));
  CS_CUDA_TRY(cudaStreamSynchronize(e->st));
  return CS_OK;
}

namespace {
int read_f32_as_f64(cs_engine* e, const float* src, size_t n, double* out) {
  std::vector<float> t(n);
  CS_CUDA_TRY(cudaStreamSynchronize(e->st));
  CS_CUDA_TRY(cudaMemcpy(t.data(), src, n * 4, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) out[i] = t[i];
  return CS_OK;
}
}  // namespace

extern "C" int cs_read_lora_grads(cs_engine* e, int layer, double* grad_a, double* grad_b) {
  if (!e || layer < 0 || layer >= e->NL) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "read_lora_grads: bad layer");
  const size_t na = (size_t)e->f * e->r, nb = (size_t)e->r * e->h;
  if (grad_a) TRY(read_f32_as_f64(e, e->gA + layer * na, na, grad_a));
  if (grad_b) TRY(read_f32_as_f64(e, e->gB + layer * nb, nb, grad_b));
  return CS_OK;
}

extern "C" int cs_read_kvgrad(cs_engine* e, int32_t L, double* dk_out, double* dv_out) {
  if (!e || L < 0 || L > e->L_max) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "read_kvgrad: bad L");
  const size_t n = (size_t)L * e->kv_dim;
  if (dk_out) TRY(read_f32_as_f64(e, e->dk_acc, n, dk_out));
  if (dv_out) TRY(read_f32_as_f64(e, e->dv_acc, n, dv_out));
  return CS_OK;
}

extern "C" int cs_read_dy(cs_engine* e, int32_t L, double* out) {
  if (!e || L < 0 || L > e->L_max || !out) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "read_dy: bad L");
  return read_f32_as_f64(e, e->dy[e->dy_cur], (size_t)L * e->h, out);
}

extern "C" int cs_read_kv(cs_engine* e, int layer, const int32_t* pages, int32_t len, double* k_out,
                          double* v_out) {
  if (!e || layer < 0 || layer >= e->NL || len < 0 || (!pages && len > 0))
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "read_kv: bad arguments");
  const size_t kv_layer = (size_t)e->npages * e->P * e->kv_dim;
  std::vector<bf16> t(e->kv_dim);
  CS_CUDA_TRY(cudaStreamSynchronize(e->st));
  for (int i = 0; i < len; ++i) {
    const int pg = pages[i / e->P];
    if (pg < 0 || pg >= e->npages) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "read_kv: page out of range");
    const size_t row = (size_t)pg * e->P + (i % e->P);
    for (int which = 0; which < 2; ++which) {
      double* o = which ? v_out : k_out;
      if (!o) continue;
      const bf16* src = (which ? e->v_pool : e->k_pool) + layer * kv_layer + row * e->kv_dim;
      CS_CUDA_TRY(cudaMemcpy(t.data(), src, e->kv_dim * sizeof(bf16), cudaMemcpyDeviceToHost));
      for (int c = 0; c < e->kv_dim; ++c) o[(size_t)i * e->kv_dim + c] = __bfloat162float(t[c]);
    }
  }
  return CS_OK;
}
