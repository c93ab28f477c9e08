// coserve/scheduler.hpp -- FlexLLM's hybrid token scheduler (§6.2).
//
//   plan_iteration        Orca iteration-level batching (max_batch, FIFO admission through
//                         MemoryModel::try_admit), chunked prefill, c = inference tokens,
//                         s = max_finetune_tokens(c, budget), attach s tokens of the active
//                         finetuning mini-batch's current phase.
//   advance_finetune      forward l += s until L -> backward at layer N-1 with l_j = L;
//                         backward l_j -= s, at 0 move to layer n-1; at layer -1 the mini-batch
//                         is done (Adam).
//   enforce_dependencies  rejects backward tokens before the forward pass completed and plans
//                         that mix two mini-batches.
// Pure host code; deterministic.  The GPU engine consumes IterationPlan through the C ABI.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <stdexcept>
#include <vector>

#include "coserve/cost_model.hpp"

namespace coserve {

struct Request {
  int64_t id = 0;
  int tenant = 0;
  int prompt_len = 1;
  int gen_len = 1;
  double arrival_ms = 0.0;
  // state
  int prefilled = 0;  // prompt tokens already processed
  int emitted = 0;    // generated tokens
  std::vector<int32_t> pages;
  double first_token_ms = -1.0;
  double completion_ms = -1.0;
  int evictions = 0;
  int32_t last_token = 0;  // next input token for decode
  double last_emit_ms = -1.0;  // time its latest token was emitted (inter-token latency)
  bool done() const { return emitted >= gen_len; }
  bool in_prefill() const { return prefilled < prompt_len; }
  int context() const { return prefilled + std::max(0, emitted - 1); }
};

enum class FtPhase : int { Idle = 0, Forward = 1, Backward = 2, Done = 3 };

struct FtState {
  int64_t minibatch = -1;
  int L = 0;
  int n_layers = 0;
  FtPhase phase = FtPhase::Idle;
  int l = 0;       // forward: tokens processed (l_i)
  int layer = 0;   // backward: current layer n
  int lj = 0;      // backward: window end l_j
  int64_t fwd_tokens = 0, bwd_tokens = 0;  // accounting
};

struct SchedulerConfig {
  int max_batch = 64;
  int chunk_size = 512;
  double tpot_slo_ms = 50.0;   // step budget = TPOT SLO
  double ttft_slo_ms = 5000.0;
  int max_tokens = 8192;       // engine capacity per iteration
  int max_ft_window = 8192;    // cap on s (multi_layer_bwd: on each backward window; an
                               // iteration may then carry several windows of one layer)
  // B200 runtime extension: one iteration may carry consecutive backward windows across
  // layers (layer n to 0, then n-1 from L) when the budget allows -- Alg. 2 order is kept.
  // false reproduces SPEC.md:433 (one layer per iteration).
  bool multi_layer_bwd = false;
  // admission done by the caller before planning (VTC fair admission, coserve/vtc.hpp)
  bool external_admission = false;
};

struct BwdWindow {
  int layer = 0;
  int lj = 0;  // window end
  int s = 0;
};

struct PrefillChunk {
  int req = 0;     // index into `running`
  int start = 0;   // first prompt position of the chunk
  int len = 0;
};

struct IterationPlan {
  std::vector<int> decode;              // indices into `running` (one token each)
  std::vector<PrefillChunk> prefill;
  int64_t c = 0;                        // inference tokens
  int64_t s = 0;                        // finetuning tokens attached
  FtPhase ft_phase = FtPhase::Idle;
  int64_t ft_minibatch = -1;
  int ft_layer = -1;                    // backward layer
  int ft_l = 0;                         // forward: l_i ; backward: l_j (window end)
  double predicted_ms = 0.0;
  std::vector<int64_t> admitted;        // request ids admitted this iteration
  std::vector<BwdWindow> bwd;           // backward windows (first = ft_layer / ft_l / s)
};

// Tokens the FT state can still take in its current phase (window clipping).
inline int64_t ft_phase_remaining(const FtState& ft) {
  if (ft.phase == FtPhase::Forward) return ft.L - ft.l;
  if (ft.phase == FtPhase::Backward) return ft.lj;
  return 0;
}

// admit FIFO while the batch has room and pages are available
inline std::vector<int64_t> admit_requests(std::deque<Request>& queue, std::vector<Request>& running,
                                           MemoryModel& mem, const SchedulerConfig& cfg) {
  std::vector<int64_t> ids;
  while (!queue.empty() && (int)running.size() < cfg.max_batch) {
    Request& r = queue.front();
    std::vector<int32_t> pages;
    if (!mem.try_admit(r.prompt_len, &pages)) break;  // FIFO: head-of-line blocks
    r.pages = std::move(pages);
    ids.push_back(r.id);
    running.push_back(std::move(r));
    queue.pop_front();
  }
  return ids;
}

// SPEC.md:421-429.  `running` holds admitted requests (prefill or decode), in admission order.
inline IterationPlan plan_iteration(std::deque<Request>& queue, std::vector<Request>& running,
                                    const FtState& ft, const LatencyProfile& prof,
                                    const SchedulerConfig& cfg, MemoryModel& mem,
                                    double budget_ms) {
  IterationPlan p;
  if (!cfg.external_admission) p.admitted = admit_requests(queue, running, mem, cfg);
  // inference rows are sized against the cost the planner charges them (inference_cost: per-row
  // decode / prefill slopes when the profile has them, latency(c, 0) otherwise -- then this is
  // exactly the spec's token budget max_finetune_tokens(prof, 0, budget)), so the inference part
  // alone never exceeds the budget whatever the fitted slopes
  int64_t n_dec = 0, n_pre = 0;
  auto fits = [&](int64_t nd, int64_t np) {
    return nd + np <= cfg.max_tokens && inference_cost(prof, nd, np) <= budget_ms;
  };
  // (1) decodes of running requests past their prompt
  for (int i = 0; i < (int)running.size(); ++i) {
    const Request& r = running[i];
    if (!r.in_prefill() && !r.done() && fits(n_dec + 1, 0)) {
      p.decode.push_back(i);
      n_dec += 1;
    }
  }
  // (2) chunked prefill in admission order within the remaining budget
  for (int i = 0; i < (int)running.size(); ++i) {
    const Request& r = running[i];
    if (!r.in_prefill()) continue;
    const int64_t room = max_tokens_within([&](int64_t x) { return fits(n_dec, n_pre + x) ? 0.0 : 1.0; },
                                           (int64_t)cfg.max_tokens - n_dec - n_pre, 0.5);
    if (room <= 0) break;
    const int len = (int)std::min<int64_t>({(int64_t)cfg.chunk_size, (int64_t)(r.prompt_len - r.prefilled), room});
    if (len <= 0) continue;
    p.prefill.push_back(PrefillChunk{i, r.prefilled, len});
    n_pre += len;
  }
  const int64_t c = n_dec + n_pre;
  p.c = c;
  // (3) s = argmax f(c, s) <= budget, clipped to the FT phase and engine capacity
  const double w_b = prof.bwd_token_weight > 0 ? prof.bwd_token_weight : 1.0;
  if (!prof.has_ctx_terms() && !cfg.multi_layer_bwd) {
    // the spec's single-profile form
    if (ft.phase == FtPhase::Forward || ft.phase == FtPhase::Backward) {
      int64_t s = max_finetune_tokens(prof, c, budget_ms);
      if (ft.phase == FtPhase::Backward && w_b != 1.0) s = (int64_t)std::floor((double)s / w_b);
      s = std::min<int64_t>(s, ft_phase_remaining(ft));
      s = std::min<int64_t>(s, cfg.max_ft_window);
      // forward rows share the engine's token capacity with the inference rows; a backward
      // window is bounded by the same capacity (engine.cu backward_window: s <= max_tokens)
      s = std::min<int64_t>(s, ft.phase == FtPhase::Forward ? cfg.max_tokens - c : (int64_t)cfg.max_tokens);
      s = std::max<int64_t>(s, 0);
      p.s = s;
      if (s > 0) {
        p.ft_phase = ft.phase;
        p.ft_minibatch = ft.minibatch;
        p.ft_layer = ft.phase == FtPhase::Backward ? ft.layer : -1;
        p.ft_l = ft.phase == FtPhase::Forward ? ft.l : ft.lj;
        if (ft.phase == FtPhase::Backward) p.bwd.push_back(BwdWindow{ft.layer, ft.lj, (int)s});
      }
    }
    const int64_t s_eq = (p.ft_phase == FtPhase::Backward && w_b != 1.0)
                             ? (int64_t)std::ceil((double)p.s * w_b) : p.s;
    p.predicted_ms = latency(prof, p.c, s_eq);
    return p;
  }
  // profile with context terms: exact argmax of the window cost within the remaining budget
  const double base = inference_cost(prof, (int64_t)p.decode.size(), c - (int64_t)p.decode.size());
  double room = budget_ms - base;
  double cost = 0.0;
  if (ft.phase == FtPhase::Forward) {
    // multi-window iterations: consecutive forward windows fuse into one segment (Alg. 2
    // windows are additive), so the window cap does not bind
    const int64_t cap = cfg.multi_layer_bwd
                            ? std::min<int64_t>((int64_t)(ft.L - ft.l), (int64_t)cfg.max_tokens - c)
                            : std::min<int64_t>({(int64_t)(ft.L - ft.l), (int64_t)cfg.max_ft_window,
                                                 (int64_t)cfg.max_tokens - c});
    const int64_t l0 = ft.l;
    const int64_t s = max_tokens_within([&](int64_t x) { return ft_fwd_cost(prof, l0, x); }, cap, room);
    if (s > 0) {
      p.s = s;
      p.ft_phase = FtPhase::Forward;
      p.ft_minibatch = ft.minibatch;
      p.ft_l = ft.l;
      cost = ft_fwd_cost(prof, l0, s);
    }
  } else if (ft.phase == FtPhase::Backward) {
    int layer = ft.layer, lj = ft.lj;
    while (layer >= 0 && room > 0) {
      const int64_t cap = std::min<int64_t>({(int64_t)lj, (int64_t)cfg.max_ft_window, (int64_t)cfg.max_tokens});  // same cap as the engine's backward_window
      const int64_t lj0 = lj;
      const int ly = layer;
      const int64_t s = max_tokens_within([&](int64_t x) { return ft_bwd_cost(prof, lj0, x, ly); }, cap, room);
      if (s <= 0) break;
      const double cw = ft_bwd_cost(prof, lj0, s, ly);
      p.bwd.push_back(BwdWindow{layer, lj, (int)s});
      p.s += s;
      cost += cw;
      room -= cw;
      lj -= (int)s;
      if (!cfg.multi_layer_bwd) break;
      if (lj > 0) {
        if (s < cap) break;  // budget-bound: the iteration is full
        continue;            // window-bound: the next window of the same layer
      }
      layer -= 1;
      lj = ft.L;
    }
    if (!p.bwd.empty()) {
      p.ft_phase = FtPhase::Backward;
      p.ft_minibatch = ft.minibatch;
      p.ft_layer = p.bwd[0].layer;
      p.ft_l = p.bwd[0].lj;
    }
  }
  p.predicted_ms = base + cost;
  return p;
}

// SPEC.md:430-438
inline void advance_finetune(FtState& ft, int64_t s) {
  if (s <= 0) return;
  if (ft.phase == FtPhase::Forward) {
    s = std::min<int64_t>(s, ft.L - ft.l);
    ft.l += (int)s;
    ft.fwd_tokens += s;
    if (ft.l >= ft.L) {
      ft.phase = FtPhase::Backward;
      ft.layer = ft.n_layers - 1;
      ft.lj = ft.L;
    }
  } else if (ft.phase == FtPhase::Backward) {
    s = std::min<int64_t>(s, ft.lj);
    ft.lj -= (int)s;
    ft.bwd_tokens += s;
    if (ft.lj == 0) {
      ft.layer -= 1;
      ft.lj = ft.L;
      if (ft.layer < 0) ft.phase = FtPhase::Done;  // optimizer step, mini-batch done
    }
  }
}

// returns false (planner bug) on a dependency violation.
inline bool enforce_dependencies(const IterationPlan& p, const FtState& ft) {
  if (p.s == 0) return true;
  if (p.ft_minibatch != ft.minibatch) return false;                    // two mini-batches
  if (p.ft_phase == FtPhase::Backward && ft.phase != FtPhase::Backward) return false;
  if (p.ft_phase == FtPhase::Backward && ft.l < ft.L) return false;    // fwd incomplete
  if (p.ft_phase == FtPhase::Forward && ft.phase != FtPhase::Forward) return false;
  return true;
}

}  // namespace coserve
