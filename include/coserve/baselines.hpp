// coserve/baselines.hpp -- the comparison policies of PAPER.md §8.2 (SPEC.md:474-548
// "baseline_schedulers"), run on the same engine and step as co-serving:
//   * temporal sharing with a fixed inference frequency n: n inference-only iterations, then
//     one finetuning iteration -- the whole mini-batch (forward windows over L tokens, the
//     backward through every layer, Adam) with inference blocked;
//   * dynamic temporal sharing (DTS, PAPER.md:528-590 Algorithm "Dynamic Temporal Sharing"):
//     the number of inference steps before the next finetuning iteration follows queue /
//     spike / backlog pressure with hysteresis and a decision delay.
//   * spatial sharing (§3 / Fig. 1(c)(d)): a fraction rho of the GPU
//     serves inference and 1 - rho finetunes, concurrently, each side slowed by the
//     interference coefficient gamma: an inference iteration takes gamma / rho of its
//     dedicated-GPU time, and in that tick the finetuning side does (1 - rho) / gamma of the
//     tick's length of dedicated-GPU finetuning work;
//   * resource isolation ("two separate memory/cost models and a static request
//     router"): the same split with no interference (gamma = 1) -- dedicated capacity for each
//     workload, nothing shared.
// The split is the spec's fractional abstraction ("no MPS/MIG modeling"): both
// sides' kernels really run on the engine, the clock charges the modelled concurrency.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

#include "coserve/cost_model.hpp"
#include "coserve/scheduler.hpp"

namespace coserve {

enum class Policy : int { Coserve = 0, TemporalFixed = 1, Dts = 2, Spatial = 3, Isolate = 4 };

// SpatialSplit: inference fraction rho in (0, 1), interference gamma >= 1
struct SpatialSplit {
  double rho = 0.5;
  double gamma = 1.15;  // SPEC.md:529 default
  double inf_factor() const { return gamma / rho; }          // inference latency multiplier
  double ft_factor() const { return (1.0 - rho) / gamma; }   // finetuning throughput multiplier
};

// DtsState (f_p initial value 64 is SPEC.md's design decision, the paper
// never initialises it)
struct DtsState {
  std::vector<double> Q, B;  // queue-length / batch-size samples since the last reset
  double r_a = 0, r_c = 0;   // arrivals / completions accumulated
  double s = 64;             // steps until the next switch to finetuning
  double f_p = 64;           // previous (smoothed) frequency
  int d = 0;                 // decision-delay counter
};

// Compute_Next_Interval
inline double dts_compute_interval(DtsState& st) {
  if (st.Q.empty()) return 64.0;
  double qsum = 0, qmax = st.Q[0];
  for (double q : st.Q) {
    qsum += q;
    qmax = std::max(qmax, q);
  }
  const double n = (double)st.Q.size();
  const double qbar = qsum / n;
  const double lambda = st.r_a / n, mu = st.r_c / n;
  const double p = std::min(1.0, qbar / 20.0) + std::min(0.5, qmax / 25.0) +
                   std::max(0.0, (lambda - mu) / 8.0);
  double f;
  if (p <= 0.8) {
    f = 64.0;
  } else if (p >= 2.0) {
    f = 512.0;
  } else {
    const double pn = (p - 0.8) / 1.2;
    f = 64.0 + pn * 0.6 * (512.0 - 64.0);
  }
  f *= 1.35;  // stabilization adjustment
  double fs = (f + 2.0 * st.f_p) / 3.0;
  st.f_p = fs;
  fs = std::max(fs, 64.0 + 16.0);
  return std::min(512.0, std::max(64.0, fs));
}

// Scheduler_Step: true -> switch to finetuning now
inline bool dts_step(DtsState& st, double q, double b, double a, double c) {
  st.r_a += a;
  st.r_c += c;
  st.Q.push_back(q);
  st.B.push_back(b);
  st.s -= 1.0;
  if (st.s <= 0.0) {
    st.d += 1;
    if (st.d >= 3) {
      st.s = dts_compute_interval(st);
      st.d = 0;
    } else {
      st.s = std::min(512.0, st.f_p * 1.1);
    }
    st.Q.clear();  // Reset_Stats
    st.B.clear();
    st.r_a = 0;
    st.r_c = 0;
    return true;
  }
  return false;
}

// One step of a temporal-sharing finetuning iteration (inference blocked): the next forward
// window (the rest of the sequence, up to the engine's token capacity) or the next backward
// window (one layer, up to the window cap).  Predicted cost = the fixed step cost plus the
// window's marginal cost from the same profile the co-serving planner uses.
inline IterationPlan plan_ft_block(const FtState& ft, const LatencyProfile& prof,
                                   const SchedulerConfig& cfg) {
  IterationPlan p;
  p.predicted_ms = inference_cost(prof, 0, 0);
  if (ft.phase == FtPhase::Forward) {
    const int64_t s = std::min<int64_t>((int64_t)(ft.L - ft.l), (int64_t)cfg.max_tokens);
    if (s <= 0) return p;
    p.s = s;
    p.ft_phase = FtPhase::Forward;
    p.ft_minibatch = ft.minibatch;
    p.ft_l = ft.l;
    p.predicted_ms += ft_fwd_cost(prof, ft.l, s);
  } else if (ft.phase == FtPhase::Backward) {
    const int64_t s = std::min<int64_t>({(int64_t)ft.lj, (int64_t)cfg.max_ft_window,
                                         (int64_t)cfg.max_tokens});
    if (s <= 0) return p;
    p.s = s;
    p.ft_phase = FtPhase::Backward;
    p.ft_minibatch = ft.minibatch;
    p.ft_layer = ft.layer;
    p.ft_l = ft.lj;
    p.bwd.push_back(BwdWindow{ft.layer, ft.lj, (int)s});
    p.predicted_ms += ft_bwd_cost(prof, ft.lj, s, ft.layer);
  }
  return p;
}

}  // namespace coserve
