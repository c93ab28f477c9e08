// coserve/gpu.hpp -- header-only C++ operator-level drop-in for the reference's hot path
// (namespace coserve, value types, exceptions), running on libcoserve_cuda.so (include/
// coserve_cuda.h).  A reference user keeps TinyModel / forward_full / backward_full and the
// spec's window API; this header gives the same calls on a B200:
//
//   reference (CPU, f64)                              here (coserve::gpu, B200)
//   TinyModel::init(cfg)            tiny_model.hpp:44  Engine::from_tiny_model(model, L_max)
//   forward_window(m, r, l_i, C)    SPEC.md:283-291    forward_window(eng, tokens, l_i, targets, C)
//   generative_loss(...)            SPEC.md:301-309      -> its return value (fused CE)
//   backward_window(m, n, ..., C,A) SPEC.md:292-300    backward_window(eng, n, l_j, s_j, C)
//   forward_full + backward_full    tiny_model.hpp:181-327  forward_backward_full(eng, tokens)
//   LoraGrads / max_grad_rel_err    tiny_model.hpp:71-92    Engine::lora_grads(l) -> HostMatrix
//   Adam once per mini-batch        SPEC.md:433,459    Engine::adam_step(...)
//
// Error conventions follow the reference: bad configs / inputs throw
// std::invalid_argument (tiny_model.hpp:45-47, matrix.hpp:70), runtime failures
// std::runtime_error; the spec's cache-desync and ordering violations throw
// CacheDesync / OrderingViolation (both std::runtime_error).  Value semantics like the
// reference: results come back as host matrices the caller owns (HostMatrix, convertible to
// the reference's coserve::Matrix with to<Matrix>()).  One host thread per Engine.
//
// Differences the device path imposes (all documented in DESIGN.md): the window's logits are
// consumed on the device by the fused cross-entropy, so forward_window returns the window's
// generative-loss sum instead of a [s, V] logits slice; graph pruning (pruning.hpp:88-172)
// means layer 0 forms no dK / dV / dX, so forward_backward_full leaves those empty.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "coserve_cuda.h"

namespace coserve {
namespace gpu {

class CacheDesync : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class OrderingViolation : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// C ABI status -> the reference's exception types
inline void check(int rc, const char* what) {
  if (rc == CS_OK) return;
  const std::string msg = std::string(what) + ": " + cs_last_error();
  switch (rc) {
    case CS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case CS_ERR_CACHE_DESYNC: throw CacheDesync(msg);
    case CS_ERR_ORDERING: throw OrderingViolation(msg);
    default: throw std::runtime_error(msg);
  }
}

// Row-major f64 host matrix (the reference Matrix's accessors: rows(), cols(), (r, c), data()).
struct HostMatrix {
  std::size_t r = 0, c = 0;
  std::vector<double> v;
  HostMatrix() = default;
  HostMatrix(std::size_t rows, std::size_t cols) : r(rows), c(cols), v(rows * cols, 0.0) {}
  std::size_t rows() const { return r; }
  std::size_t cols() const { return c; }
  bool empty() const { return v.empty(); }
  double& operator()(std::size_t i, std::size_t j) { return v[i * c + j]; }
  double operator()(std::size_t i, std::size_t j) const { return v[i * c + j]; }
  const std::vector<double>& data() const { return v; }
  std::vector<double>& data() { return v; }
  // copy into any matrix type with (rows, cols) construction and data() (coserve::Matrix)
  template <class MatrixT>
  MatrixT to() const {
    MatrixT m(r, c);
    for (std::size_t i = 0; i < v.size(); ++i) m.data()[i] = v[i];
    return m;
  }
};

// SPEC.md:248-252 for the finetuning sequence.  The Q/K/V rows live in the engine's paged pools
// (device memory); the host side is the sequence's page table and its current length.
struct QkvCache {
  std::vector<int32_t> pages;
  int seq_len = 0;
  int length = 0;
};

class Engine {
 public:
  explicit Engine(const cs_model_config& cfg, int device = 0) : cfg_(cfg) {
    check(cs_engine_create(&cfg_, device, 0, 1, nullptr, &e_), "cs_engine_create");
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&& o) noexcept : cfg_(o.cfg_), e_(std::exchange(o.e_, nullptr)) {}
  Engine& operator=(Engine&& o) noexcept {
    if (this != &o) {
      reset();
      cfg_ = o.cfg_;
      e_ = std::exchange(o.e_, nullptr);
    }
    return *this;
  }
  ~Engine() { reset(); }

  cs_engine* get() const { return e_; }
  const cs_model_config& config() const { return cfg_; }

  // weights in the reference layout: row-major [in, out] (tiny_model.hpp:31-35)
  void set_weight(const char* name, int layer, const double* data, std::size_t rows, std::size_t cols) {
    check(cs_engine_set_weight(e_, name, layer, data, 0, (int64_t)rows, (int64_t)cols), name);
  }
  template <class MatrixT>
  void set_weight(const char* name, int layer, const MatrixT& m) {
    set_weight(name, layer, m.data().data(), m.rows(), m.cols());
  }

  // TinyModel::init-compatible construction (tiny_model.hpp:17-67): the reference model's
  // frozen weights and LoRA adapters, uploaded (bf16 frozen copies, fp32 LoRA masters).
  // TinyModelT is the reference's coserve::TinyModel (or anything with its members).
  template <class TinyModelT>
  static Engine from_tiny_model(const TinyModelT& m, int max_ft_len, int device = 0,
                                int max_tokens = 0, int page_size = 16, int n_pages = 0) {
    cs_model_config c{};
    c.n_layers = m.cfg.depth;
    c.hidden = (int32_t)m.cfg.hidden;
    c.n_heads = m.cfg.heads;
    c.n_kv_heads = m.cfg.heads;
    if (m.cfg.heads < 1 || m.cfg.hidden % m.cfg.heads != 0)
      throw std::invalid_argument("tiny model: heads must divide hidden");  // tiny_model.hpp:45
    c.head_dim = (int32_t)(m.cfg.hidden / m.cfg.heads);
    c.ffn = (int32_t)(m.cfg.hidden * m.cfg.ffn_mult);
    c.vocab = (int32_t)m.cfg.vocab;
    c.lora_rank = m.cfg.lora_rank;
    c.norm = 0;
    c.act = 0;
    c.rope = 0;
    c.qkv_bias = 0;
    c.rope_theta = 10000.f;
    c.rms_eps = 1e-5f;
    c.page_size = page_size;
    c.max_ft_len = max_ft_len;
    c.max_tokens = max_tokens > 0 ? max_tokens : max_ft_len;
    c.n_pages = n_pages > 0 ? n_pages : (max_ft_len + page_size - 1) / page_size + 8;
    c.max_segments = 8;
    Engine e(c, device);
    e.set_weight("embed", 0, m.embed);
    e.set_weight("unembed", 0, m.unembed);
    for (int l = 0; l < (int)m.layers.size(); ++l) {
      const auto& w = m.layers[l];
      e.set_weight("wq", l, w.wq);
      e.set_weight("wk", l, w.wk);
      e.set_weight("wv", l, w.wv);
      e.set_weight("wo", l, w.wo);
      e.set_weight("w_up", l, w.w_up);
      e.set_weight("w_down", l, w.w_down);
      e.set_weight("lora_a", l, w.lora_a);
      e.set_weight("lora_b", l, w.lora_b);
    }
    return e;
  }

  // LoraGrads (tiny_model.hpp:71-83) of one layer: dA [f, r], dB [r, h]
  std::pair<HostMatrix, HostMatrix> lora_grads(int layer) const {
    HostMatrix a(cfg_.ffn, cfg_.lora_rank), b(cfg_.lora_rank, cfg_.hidden);
    check(cs_read_lora_grads(e_, layer, a.v.data(), b.v.data()), "cs_read_lora_grads");
    return {std::move(a), std::move(b)};
  }
  // LoRA master weights (fp32 on the device), e.g. after adam_step
  std::pair<HostMatrix, HostMatrix> lora(int layer) const {
    HostMatrix a(cfg_.ffn, cfg_.lora_rank), b(cfg_.lora_rank, cfg_.hidden);
    check(cs_engine_get_lora(e_, layer, a.v.data(), b.v.data()), "cs_engine_get_lora");
    return {std::move(a), std::move(b)};
  }
  // Adam once per mini-batch, after the last backward window
  void adam_step(float lr = 1e-3f, float beta1 = 0.9f, float beta2 = 0.999f, float eps = 1e-8f) {
    check(cs_adam_step(e_, lr, beta1, beta2, eps), "cs_adam_step");
  }
  void reset_finetuning() { check(cs_engine_reset_ft(e_), "cs_engine_reset_ft"); }

  // a cache for a finetuning sequence of seq_len tokens on pages [first_page, ...)
  QkvCache make_cache(int seq_len, int first_page = 0) const {
    if (seq_len < 1 || seq_len > cfg_.max_ft_len)
      throw std::invalid_argument("make_cache: seq_len must be in [1, max_ft_len]");
    QkvCache c;
    c.seq_len = seq_len;
    const int n = (seq_len + cfg_.page_size - 1) / cfg_.page_size;
    if (first_page < 0 || first_page + n > cfg_.n_pages)
      throw std::invalid_argument("make_cache: not enough KV pages");
    for (int i = 0; i < n; ++i) c.pages.push_back(first_page + i);
    return c;
  }

 private:
  void reset() {
    if (e_) cs_engine_destroy(e_);
    e_ = nullptr;
  }
  cs_model_config cfg_{};
  cs_engine* e_ = nullptr;
};

// forward_window: the window's tokens at positions [l_i, l_i + s) through all
// layers, attending to the cached [0, l_i); appends Q, K, V.  targets[i] is the next-token id of
// row i (-1: none, the sequence's last row).  Returns the window's summed next-token CE
// (generative_loss); divide the sum over all windows by (L - 1) once.
inline double forward_window(Engine& e, const std::vector<int>& tokens_window, int l_i,
                             const std::vector<int>& targets, QkvCache& cache) {
  const int s = (int)tokens_window.size();
  if (s < 1) throw std::invalid_argument("forward_window: empty window");
  if ((int)targets.size() != s) throw std::invalid_argument("forward_window: one target per token");
  if (cache.length != l_i)
    throw CacheDesync("forward_window: cache length " + std::to_string(cache.length) +
                      " != l_i " + std::to_string(l_i));
  if (l_i + s > cache.seq_len) throw std::invalid_argument("forward_window: window past the sequence");
  std::vector<int32_t> tok(tokens_window.begin(), tokens_window.end());
  std::vector<int32_t> tg(targets.begin(), targets.end());
  cs_segment seg{};
  seg.kind = CS_SEG_FT_FWD;
  seg.q_start = 0;
  seg.q_len = s;
  seg.ctx_start = l_i;
  seg.page_off = 0;
  seg.n_pages = (int32_t)cache.pages.size();
  seg.sample = 0;
  seg.adapter = 1;
  cs_iteration_plan p{};
  p.n_tokens = s;
  p.tokens = tok.data();
  p.n_segments = 1;
  p.segments = &seg;
  p.page_table = cache.pages.data();
  p.page_table_len = (int32_t)cache.pages.size();
  p.ft.phase = CS_FT_FORWARD;
  p.ft.seq_len = cache.seq_len;
  p.ft.l = l_i;
  p.ft.s = s;
  p.ft.targets = tg.data();
  cs_step_result r{};
  check(cs_step(e.get(), &p, &r), "forward_window");
  cache.length = l_i + s;
  return r.ft_loss_sum;
}

// forward_window over a sequence: targets from the sequence itself (token i+1, -1 for the last)
inline double forward_window(Engine& e, const std::vector<int>& sequence, int l_i, int s, QkvCache& cache) {
  if (l_i < 0 || s < 1 || l_i + s > (int)sequence.size())
    throw std::invalid_argument("forward_window: window outside the sequence");
  std::vector<int> w(sequence.begin() + l_i, sequence.begin() + l_i + s), tg(s);
  for (int i = 0; i < s; ++i) tg[i] = l_i + i + 1 < (int)sequence.size() ? sequence[l_i + i + 1] : -1;
  return forward_window(e, w, l_i, tg, cache);
}

// backward_window: layer n, rows [l_j - s_j, l_j); windows run layer by
// layer from the top, each layer's windows in descending order (OrderingViolation otherwise).
// The engine keeps dY, ΔKVAccum and the LoRA gradients on the device.
inline void backward_window(Engine& e, int n, int l_j, int s_j, QkvCache& cache) {
  if (cache.length != cache.seq_len)
    throw OrderingViolation("backward_window: the forward pass has not completed");
  cs_iteration_plan p{};
  p.page_table = cache.pages.data();
  p.page_table_len = (int32_t)cache.pages.size();
  p.ft.phase = CS_FT_BACKWARD;
  p.ft.seq_len = cache.seq_len;
  p.ft.l = l_j;
  p.ft.s = s_j;
  p.ft.layer = n;
  p.ft.page_off = 0;
  p.ft.n_pages = (int32_t)cache.pages.size();
  cs_step_result r{};
  check(cs_step(e.get(), &p, &r), "backward_window");
}

// tiny_model.hpp:248-327 result types on the GPU path
struct GpuLayerGrads {
  HostMatrix dk, dv, dx;  // [L, h]; empty for layer 0 (pruned: no attention backward, no dX)
};
struct GpuResult {
  double loss = 0.0;
  std::vector<HostMatrix> grad_a, grad_b;
  std::vector<GpuLayerGrads> layers;
};

// forward_full + backward_full (tiny_model.hpp:181-327) as token-level windows on the GPU:
// forward windows of fwd_window tokens, backward windows of bwd_window tokens (0 = whole
// sequence), then the LoRA gradients and per-layer ΔKVAccum / dX read back.
inline GpuResult forward_backward_full(Engine& e, const std::vector<int>& tokens, int fwd_window = 0,
                                       int bwd_window = 0) {
  const int L = (int)tokens.size();
  if (L < 1) throw std::invalid_argument("forward_full: empty sequence");  // tiny_model.hpp:183
  e.reset_finetuning();
  QkvCache cache = e.make_cache(L);
  const int fw = fwd_window > 0 ? fwd_window : L;
  const int bw = bwd_window > 0 ? bwd_window : L;
  GpuResult out;
  double loss_sum = 0.0;
  for (int l = 0; l < L; l += fw) loss_sum += forward_window(e, tokens, l, std::min(fw, L - l), cache);
  out.loss = L > 1 ? loss_sum / (double)(L - 1) : 0.0;
  const cs_model_config& c = e.config();
  const int kv = c.n_kv_heads * c.head_dim;
  out.layers.resize(c.n_layers);
  for (int n = c.n_layers - 1; n >= 0; --n) {
    for (int lj = L; lj > 0; lj -= std::min(bw, lj)) backward_window(e, n, lj, std::min(bw, lj), cache);
    if (n > 0) {
      GpuLayerGrads g{HostMatrix(L, kv), HostMatrix(L, kv), HostMatrix(L, c.hidden)};
      check(cs_read_kvgrad(e.get(), L, g.dk.v.data(), g.dv.v.data()), "cs_read_kvgrad");
      check(cs_read_dy(e.get(), L, g.dx.v.data()), "cs_read_dy");
      out.layers[n] = std::move(g);
    }
  }
  for (int l = 0; l < c.n_layers; ++l) {
    auto ab = e.lora_grads(l);
    out.grad_a.push_back(std::move(ab.first));
    out.grad_b.push_back(std::move(ab.second));
  }
  return out;
}

}  // namespace gpu
}  // namespace coserve
