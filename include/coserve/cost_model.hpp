// coserve/cost_model.hpp -- latency estimation f(c, s), its exact inverse, and the paged-KV
// memory model with admission control (§6.2, §7).
// Header-only host C++ (namespace coserve, like the reference's proj/include/coserve/).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <vector>

namespace coserve {

// f is strictly increasing in c+s; f(0,0) = t0 > 0.
struct LatencyProfile {
  double t0_ms = 2.0;
  double slope_ms_per_token = 0.01;
  double knee_tokens = std::numeric_limits<double>::infinity();  // slope doubles past the knee
  // Cost of one backward-window token relative to a forward token.  SPEC.md:458 charges both
  // through the same f (weight 1, the default); a measured B200 profile sets it from the
  // offline profiler (a backward token touches one layer, a forward token all of them).
  double bwd_token_weight = 1.0;
  // Attention's context dependence (B200 profile; 0 = the spec's f(c, s)): a forward window
  // of s tokens at position l costs an extra attn_fwd * s * (l + s/2); a backward window ending
  // at l_j costs an extra attn_bwd * s * (l_j - s/2).
  double attn_fwd_ms_per_token_ctx = 0.0;
  double attn_bwd_ms_per_token_ctx = 0.0;
  // cost of a layer-0 backward window relative to another layer's (graph pruning leaves only
  // the MLP/LoRA part there); 1 = no distinction
  double bwd_layer0_weight = 1.0;
  // Inference rows are not finetuning rows (no loss head, no saved activations): a measured
  // profile charges decode rows and prefill tokens their own slopes (0 = the common slope).
  double decode_ms_per_row = 0.0;
  double prefill_ms_per_token = 0.0;
  // Fixed cost of a finetuning forward window (its loss head / CE / saved-activation launches,
  // independent of s); 0 = none.  Without it the per-token slope absorbs it and small windows
  // (the tail of a sequence, at long context) are under-predicted.
  double fwd_window_ms = 0.0;
  bool has_ctx_terms() const { return attn_fwd_ms_per_token_ctx > 0 || attn_bwd_ms_per_token_ctx > 0; }
  bool has_row_terms() const { return decode_ms_per_row > 0 || prefill_ms_per_token > 0; }
};

// Base cost of an iteration's inference rows (n_dec decode rows + n_pre prefill tokens); equals
// latency(p, n_dec + n_pre, 0) unless the profile has per-kind row slopes.
inline double inference_cost(const LatencyProfile& p, int64_t n_dec, int64_t n_pre);

// t0 + b*min(c+s, k) + 2b*max(0, c+s-k)
inline double latency(const LatencyProfile& p, int64_t c, int64_t s) {
  if (c < 0 || s < 0) throw std::invalid_argument("latency: c, s must be >= 0");
  const double n = (double)c + (double)s;
  const double k = p.knee_tokens;
  return p.t0_ms + p.slope_ms_per_token * std::min(n, k) +
         2.0 * p.slope_ms_per_token * std::max(0.0, n - k);
}

// largest integer s >= 0 with latency(c, s) <= budget; 0 if none.
// Closed-form guess, then exact correction against latency() itself (boundary inclusive).
inline int64_t max_finetune_tokens(const LatencyProfile& p, int64_t c, double slo_step_ms) {
  if (!(slo_step_ms > 0)) throw std::invalid_argument("max_finetune_tokens: budget must be > 0");
  if (latency(p, c, 0) > slo_step_ms) return 0;
  const double b = p.slope_ms_per_token, k = p.knee_tokens;
  double n;  // total tokens allowed
  const double rem = slo_step_ms - p.t0_ms;
  if (b <= 0) return std::numeric_limits<int32_t>::max();
  if (rem / b <= k) n = rem / b;
  else n = k + (rem - b * k) / (2.0 * b);
  int64_t s = std::max<int64_t>(0, (int64_t)std::floor(n) - c);
  while (s > 0 && latency(p, c, s) > slo_step_ms) --s;
  while (latency(p, c, s + 1) <= slo_step_ms) ++s;
  return s;
}

inline double inference_cost(const LatencyProfile& p, int64_t n_dec, int64_t n_pre) {
  if (!p.has_row_terms()) return latency(p, n_dec + n_pre, 0);
  const double d = p.decode_ms_per_row > 0 ? p.decode_ms_per_row : p.slope_ms_per_token;
  const double f = p.prefill_ms_per_token > 0 ? p.prefill_ms_per_token : p.slope_ms_per_token;
  return p.t0_ms + d * (double)n_dec + f * (double)n_pre;
}

// Marginal cost of finetuning windows on top of latency(c, 0) (profile with context terms).
inline double ft_fwd_cost(const LatencyProfile& p, int64_t l, int64_t s) {
  return (s > 0 ? p.fwd_window_ms : 0.0) + p.slope_ms_per_token * (double)s +
         p.attn_fwd_ms_per_token_ctx * (double)s * ((double)l + 0.5 * (double)s);
}
inline double ft_bwd_cost(const LatencyProfile& p, int64_t lj, int64_t s, int layer = 1) {
  const double w = p.bwd_token_weight > 0 ? p.bwd_token_weight : 1.0;
  const double c = w * p.slope_ms_per_token * (double)s +
                   p.attn_bwd_ms_per_token_ctx * (double)s * ((double)lj - 0.5 * (double)s);
  return layer == 0 ? p.bwd_layer0_weight * c : c;
}
// largest s in [0, cap] with cost(s) <= room for a cost monotone in s (binary search)
template <typename F>
inline int64_t max_tokens_within(F cost, int64_t cap, double room) {
  if (cap <= 0 || room <= 0 || cost(1) > room) return 0;
  int64_t lo = 1, hi = cap;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (cost(mid) <= room) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// pages of page_size tokens; a request is admitted iff
// ceil(prompt/page) + growth pages are free; pages are reserved atomically.
class MemoryModel {
 public:
  MemoryModel(int64_t total_pages, int64_t page_size, int64_t growth_tokens = 0)
      : total_(total_pages), page_(page_size), growth_(growth_tokens) {
    if (total_pages < 0 || page_size < 1) throw std::invalid_argument("MemoryModel: bad sizes");
    free_.reserve(total_pages);
    for (int64_t i = total_pages - 1; i >= 0; --i) free_.push_back((int32_t)i);
  }
  int64_t page_size() const { return page_; }
  int64_t free_pages() const { return (int64_t)free_.size(); }
  int64_t total_pages() const { return total_; }
  int64_t pages_for(int64_t tokens) const { return (tokens + page_ - 1) / page_; }

  // try_admit: reserve ceil(prompt/page) + ceil(growth/page) pages; returns page ids or empty
  bool try_admit(int64_t prompt_tokens, std::vector<int32_t>* pages_out) {
    const int64_t need = pages_for(prompt_tokens) + pages_for(growth_);
    if (need > free_pages() || prompt_tokens < 0) return false;
    if (pages_out) {
      pages_out->clear();
      for (int64_t i = 0; i < need; ++i) {
        pages_out->push_back(free_.back());
        free_.pop_back();
      }
    } else {
      free_.resize(free_.size() - need);
    }
    return true;
  }
  // grow a sequence by one page (decode past its reservation); false = would need eviction
  bool grow(std::vector<int32_t>* pages) {
    if (free_.empty()) return false;
    pages->push_back(free_.back());
    free_.pop_back();
    return true;
  }
  void release(const std::vector<int32_t>& pages) {
    for (auto it = pages.rbegin(); it != pages.rend(); ++it) free_.push_back(*it);
  }
  // raw reservation (finetuning sequence cache pages are not admission-controlled)
  bool reserve(int64_t n, std::vector<int32_t>* pages_out) {
    if (n > free_pages()) return false;
    for (int64_t i = 0; i < n; ++i) {
      pages_out->push_back(free_.back());
      free_.pop_back();
    }
    return true;
  }

 private:
  int64_t total_, page_, growth_;
  std::vector<int32_t> free_;  // LIFO free list: deterministic page ids
};

}  // namespace coserve
