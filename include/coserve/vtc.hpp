// coserve/vtc.hpp -- Virtual Token Counter fair co-serving (SPEC.md "fairness_vtc", PAPER.md
// Appendix C): per-tenant counters of weighted service, counter lifting on (re)arrival,
// min-counter request selection, weighted charges for prompt (w_p), generated (w_q) and
// finetuning (w_r) tokens.  Wraps the hybrid scheduler: VTC picks which tenant's queued
// request is admitted next; the token scheduler still sizes the finetuning window.
// Defaults w_p = 1, w_q = 2, w_r = 1 (SPEC.md design decision; the paper fixes no values).
#pragma once
#include <algorithm>
#include <cstdint>
#include <deque>
#include <vector>

#include "coserve/scheduler.hpp"

namespace coserve {

struct VtcLedger {
  double w_p = 1.0, w_q = 2.0, w_r = 1.0;
  std::vector<double> counter;   // c_i
  std::vector<double> service;   // W_i: cumulative weighted service
  std::vector<int> queued;       // queued requests per tenant
  double c_last = 0.0;           // counter of the last tenant whose queue emptied

  void ensure(int t) {
    if ((int)counter.size() <= t) {
      counter.resize(t + 1, 0.0);
      service.resize(t + 1, 0.0);
      queued.resize(t + 1, 0);
    }
  }
  bool any_queued() const {
    for (int q : queued)
      if (q > 0) return true;
    return false;
  }
  // on_arrival (Appendix C: c_u <- max{c_u, min{c_i | i in Q}}; empty system -> c_l)
  void on_arrival(int u) {
    ensure(u);
    if (queued[u] == 0) {
      if (!any_queued()) {
        counter[u] = std::max(counter[u], c_last);
      } else {
        double mn = 0.0;
        bool first = true;
        for (int i = 0; i < (int)queued.size(); ++i)
          if (queued[i] > 0 && (first || counter[i] < mn)) mn = counter[i], first = false;
        counter[u] = std::max(counter[u], mn);
      }
    }
    queued[u] += 1;
  }
  // select_next: the queued request of the min-counter tenant (tie: lowest tenant id), FIFO
  // within a tenant; -1 if the queue is empty
  int select(const std::deque<Request>& queue) const {
    int best = -1, best_t = 0;
    double best_c = 0.0;
    for (int i = 0; i < (int)queue.size(); ++i) {
      const int t = queue[i].tenant;
      const double c = t < (int)counter.size() ? counter[t] : 0.0;
      if (best < 0 || c < best_c || (c == best_c && t < best_t)) best = i, best_t = t, best_c = c;
    }
    return best;  // the first queued request of the chosen tenant (FIFO within it)
  }
  void charge(int u, double w_tokens) {
    ensure(u);
    counter[u] += w_tokens;
    service[u] += w_tokens;
  }
  void on_admit(int u, int prompt_len) {
    ensure(u);
    queued[u] -= 1;
    charge(u, w_p * prompt_len);
    if (queued[u] == 0) c_last = counter[u];
  }
  // Lemma 1 invariant: spread of counters over tenants with queued requests
  double queued_spread() const {
    double mn = 0, mx = 0;
    bool first = true;
    for (int i = 0; i < (int)queued.size(); ++i)
      if (queued[i] > 0) {
        if (first) mn = mx = counter[i], first = false;
        mn = std::min(mn, counter[i]);
        mx = std::max(mx, counter[i]);
      }
    return first ? 0.0 : mx - mn;
  }
};

// Admission under VTC: fill the batch with the min-counter tenant's oldest queued request
// while its KV pages fit (a blocked selection stops admission this iteration, as FIFO does)
inline std::vector<int64_t> admit_requests_vtc(std::deque<Request>& queue, std::vector<Request>& running,
                                               MemoryModel& mem, const SchedulerConfig& cfg,
                                               VtcLedger& vtc) {
  std::vector<int64_t> ids;
  while (!queue.empty() && (int)running.size() < cfg.max_batch) {
    const int i = vtc.select(queue);
    Request& r = queue[i];
    std::vector<int32_t> pages;
    if (!mem.try_admit(r.prompt_len, &pages)) break;
    r.pages = std::move(pages);
    ids.push_back(r.id);
    vtc.on_admit(r.tenant, r.prompt_len);
    running.push_back(std::move(r));
    queue.erase(queue.begin() + i);
  }
  return ids;
}

}  // namespace coserve
