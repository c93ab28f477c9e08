// coserve/coserve_loop.hpp -- the co-serving engine loop (SPEC.md:675-728 sim_engine, run on a
// real GPU): inject arrivals with time <= now, plan_iteration, execute the step, advance
// request and finetuning state, Adam at the end of each mini-batch, record metrics.
//
// The clock is either the executor's measured iteration time (GPU: wall time of the step,
// so arrivals, TTFT and TPOT are real) or the scheduler's predicted latency (simulation,
// SPEC.md:450 "charges the predicted latency") -- the latter makes plans bit-reproducible
// for parity against the oracle.  Header-only, no CUDA dependency: the GPU enters through
// the StepExecutor interface (implemented over the C ABI in csrc/coserve_run.cpp).
#pragma once
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <deque>
#include <vector>

#include "coserve/baselines.hpp"
#include "coserve/calibrate.hpp"
#include "coserve/vtc.hpp"
#include "coserve/cost_model.hpp"
#include "coserve/scheduler.hpp"
#include "coserve/workload.hpp"

namespace coserve {

struct StepSegment {
  int kind = 0;  // 0 decode, 1 prefill, 2 finetuning forward window
  std::vector<int32_t> tokens;
  int ctx_start = 0;
  const std::vector<int32_t>* pages = nullptr;
  bool sample = false;
  bool adapter = false;
};

struct StepInput {
  std::vector<StepSegment> segs;
  FtPhase ft_phase = FtPhase::Idle;
  int ft_L = 0, ft_l = 0, ft_s = 0, ft_layer = -1;
  std::vector<int32_t> ft_targets;
  const std::vector<int32_t>* ft_pages = nullptr;
  std::vector<BwdWindow> extra_bwd;  // further backward windows after (ft_layer, ft_l, ft_s)
  // wall clock at the end of the previous step: an executor's clock advance covers the whole
  // cycle -- the loop's own admission / planning / bookkeeping and the Adam step included
  std::chrono::steady_clock::time_point cycle_begin{};
};

struct StepOutput {
  std::vector<int32_t> next_tokens;  // per segment (-1 unsampled)
  double ms = 0.0;                   // clock advance
  double device_ms = 0.0;            // device time of the step
  std::chrono::steady_clock::time_point t_end{};  // wall clock when the step returned
};

class StepExecutor {
 public:
  virtual ~StepExecutor() = default;
  virtual bool run(const StepInput& in, StepOutput& out) = 0;
  virtual bool adam() = 0;
};

struct LoopConfig {
  SchedulerConfig sched;
  LatencyProfile prof;
  double budget_ms = 50.0;      // per-iteration latency budget handed to the planner
  int n_layers = 2;
  int vocab = 64;
  int page_size = 16;
  int64_t total_pages = 4096;
  int growth_tokens = 128;      // admission reservation for generation
  int ft_seq_len = 64;          // finetuning sequence length L (<= 8192)
  int warmup_iters = 0;
  int timed_iters = 100;
  int prepopulate = 0;          // requests already decoding at t=0 (steady-state start)
  bool adaptive = false;        // correct the profile with measured/predicted ratios
  // adaptive + co-serving policy + a profile with row and context terms: calibrate each
  // coefficient of f(c, s) online (coserve/calibrate.hpp) instead of one ratio per FT phase
  bool calibrate = false;
  // tail control (adaptive only; 0 = off): the planner budget becomes
  // tail_target x TPOT SLO / q95(measured / predicted over the last 96 inference iterations),
  // so the iteration-latency tail -- not the mean -- sits at the SLO on any box
  double tail_target = 0.0;
  uint64_t seed = 0;
  // scheduling policy (§8.2 baselines, coserve/baselines.hpp): co-serving, or
  // temporal sharing -- inference-only iterations interleaved with whole finetuning
  // iterations, after temporal_n inference iterations (fixed) or when DTS says so
  Policy policy = Policy::Coserve;
  int temporal_n = 128;
  SpatialSplit split;           // Policy::Spatial / Isolate (Isolate forces gamma = 1)
  bool sim_clock = false;       // advance the clock by predicted latency even with an executor
  // Virtual Token Counter fair admission across tenants (coserve/vtc.hpp, App. C);
  // finetuning tokens are charged to ft_tenant (-1: to nobody)
  bool vtc = false;
  double vtc_wp = 1.0, vtc_wq = 2.0, vtc_wr = 1.0;
  int ft_tenant = -1;
  WorkloadConfig workload;
};

struct IterLog {
  double t_ms = 0, pred_ms = 0, ms = 0, device_ms = 0;
  int c = 0, s = 0, phase = 0, layer = -1, l = 0;
  int n_decode = 0, n_prefill = 0, n_running = 0, n_queue = 0;
  bool timed = false;
};

struct LoopStats {
  int64_t iters = 0;
  double timed_ms = 0, timed_device_ms = 0;
  int64_t ft_fwd_tokens = 0, ft_bwd_tokens = 0;      // timed region
  double ft_fwd_ms = 0, ft_bwd_ms = 0;                // timed time in fwd / bwd-phase iterations
  int64_t minibatches_done = 0;                       // timed region
  int64_t inf_tokens = 0;                             // timed region (decode + prefill)
  int64_t gen_tokens = 0;
  int64_t requests_done = 0, requests_slo_ok = 0;
  int64_t evictions = 0;
  std::vector<double> ttft_ms, tpot_ms;
  // observable in short runs: the gap between consecutive tokens of every decoding request in
  // the timed region (prepopulated requests included), and SLO attainment over the requests
  // that ARRIVED in the timed region only -- completed ones by their TTFT / TPOT, unfinished ones
  // a miss once their wait for the first token already exceeds the TTFT SLO
  std::vector<double> itl_ms;
  int64_t timed_arrivals = 0, timed_done = 0, timed_slo_ok = 0, timed_unfinished_miss = 0;
  std::vector<IterLog> log;
  bool ok = true;
  // VTC: cumulative weighted service and completed requests per tenant, max spread of the
  // queued tenants' counters (Lemma 1), max |W_0 - W_1| gap over intervals where tenants 0
  // and 1 are both backlogged (Theorem 1)
  std::vector<double> tenant_service;
  std::vector<int64_t> tenant_done;
  double vtc_spread_max = 0.0, vtc_pair_gap_max = 0.0;
};

// deterministic synthetic token ids (data: synthetic)
inline int32_t synth_token(int64_t id, int64_t pos, int vocab) {
  uint64_t x = (uint64_t)id * 0x9E3779B97F4A7C15ull ^ (uint64_t)(pos + 1) * 0xBF58476D1CE4E5B9ull;
  x ^= x >> 31;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 29;
  return (int32_t)(x % (uint64_t)vocab);
}

inline LoopStats run_coserve(const LoopConfig& cfg, StepExecutor* exec) {
  LoopStats st;
  MemoryModel mem(cfg.total_pages, cfg.page_size, cfg.growth_tokens);
  const std::vector<Arrival> trace = generate_trace(cfg.workload, cfg.seed);
  size_t next_arrival = 0;
  std::deque<Request> queue;
  std::vector<Request> running;
  int64_t next_id = 0;
  double now = 0.0;
  // finetuning: one active mini-batch; its cache pages are reserved for the whole run
  FtState ft;
  ft.L = cfg.ft_seq_len;
  ft.n_layers = cfg.n_layers;
  std::vector<int32_t> ft_pages;
  std::vector<int32_t> ft_tokens;
  if (ft.L > 0) {
    if (!mem.reserve(mem.pages_for(ft.L), &ft_pages)) {
      st.ok = false;
      return st;
    }
    ft.phase = FtPhase::Forward;
    ft.minibatch = 0;
    for (int i = 0; i < ft.L; ++i) ft_tokens.push_back(synth_token(-1, i, cfg.vocab));
  }
  // steady-state start: requests already decoding (synthetic KV contents)
  {
    TraceRng prng(cfg.seed ^ 0x5EED5EEDull);
    for (int i = 0; i < cfg.prepopulate && (int)running.size() < cfg.sched.max_batch; ++i) {
      Request r;
      r.id = next_id++;
      r.prompt_len = clip_len(prng.lognormal(cfg.workload.prompt_mu, cfg.workload.prompt_sigma),
                              cfg.workload.prompt_min, cfg.workload.prompt_max);
      r.gen_len = clip_len(prng.lognormal(cfg.workload.gen_mu, cfg.workload.gen_sigma),
                           cfg.workload.gen_min, cfg.workload.gen_max);
      r.prefilled = r.prompt_len;
      r.emitted = 1 + (int)prng.uniform_int(0, std::max(0, r.gen_len - 2));
      r.arrival_ms = -1e18;  // excluded from SLO statistics
      r.first_token_ms = -1e18;
      std::vector<int32_t> pages;
      if (!mem.reserve(mem.pages_for(r.context() + 1 + cfg.growth_tokens), &pages)) break;
      r.pages = std::move(pages);
      r.last_token = synth_token(r.id, r.context(), cfg.vocab);
      running.push_back(std::move(r));
    }
  }
  double corr[3] = {1.0, 1.0, 1.0};  // adaptive, per FT phase (none / forward / backward)
  const bool use_cal = cfg.adaptive && cfg.calibrate && cfg.policy == Policy::Coserve &&
                       CostCalibrator::applicable(cfg.prof);
  CostCalibrator cal(cfg.prof);
  const bool spatial = cfg.policy == Policy::Spatial || cfg.policy == Policy::Isolate;
  const bool temporal = cfg.policy == Policy::TemporalFixed || cfg.policy == Policy::Dts;
  SpatialSplit split = cfg.split;
  if (cfg.policy == Policy::Isolate) split.gamma = 1.0;
  DtsState dts;
  VtcLedger vtc;
  vtc.w_p = cfg.vtc_wp;
  vtc.w_q = cfg.vtc_wq;
  vtc.w_r = cfg.vtc_wr;
  SchedulerConfig sched = cfg.sched;
  sched.external_admission = cfg.vtc;
  bool pair_on = false;  // tenants 0 and 1 both backlogged
  double pair_lo = 0.0, pair_hi = 0.0;
  int inf_since_ft = 0;   // inference-only iterations since the last finetuning iteration
  bool ft_block = false;  // temporal sharing: inside a finetuning iteration (inference blocked)
  std::vector<double> resid;  // ring of measured / predicted (tail control)
  size_t resid_pos = 0;
  double budget = cfg.budget_ms;
  const int total_iters = cfg.warmup_iters + cfg.timed_iters;
  auto cycle_t = std::chrono::steady_clock::now();
  double timed_t0 = 1e300;  // clock time the timed region starts
  for (int it = 0; it < total_iters; ++it) {
    const bool timed = it >= cfg.warmup_iters;
    if (timed && timed_t0 > 1e299) timed_t0 = now;
    int64_t arrived = 0;
    while (next_arrival < trace.size() && trace[next_arrival].time_ms <= now) {
      ++arrived;
      const Arrival& a = trace[next_arrival++];
      Request r;
      r.id = next_id++;
      r.tenant = a.tenant;
      r.prompt_len = a.prompt_len;
      r.gen_len = a.gen_len;
      r.arrival_ms = a.time_ms;
      if (timed && r.arrival_ms >= timed_t0) st.timed_arrivals += 1;
      if (cfg.vtc) vtc.on_arrival(r.tenant);
      queue.push_back(std::move(r));
    }
    // decode growth: make room for each decoding request's next token (eviction if none)
    for (size_t i = 0; i < running.size();) {
      Request& r = running[i];
      if (!r.in_prefill() && !r.done() &&
          (int64_t)(r.context() + 1) > (int64_t)r.pages.size() * cfg.page_size) {
        if (!mem.grow(&r.pages)) {
          mem.release(r.pages);
          r.pages.clear();
          r.prefilled = 0;
          r.emitted = 0;
          r.evictions += 1;
          st.evictions += 1;
          if (cfg.vtc) vtc.on_arrival(r.tenant);
          queue.push_front(std::move(r));
          running.erase(running.begin() + i);
          continue;
        }
      }
      ++i;
    }
    LatencyProfile prof = cfg.prof;
    const int cph = ft.phase == FtPhase::Forward ? 1 : (ft.phase == FtPhase::Backward ? 2 : 0);
    if (use_cal) {
      prof = cal.profile();
    } else if (cfg.adaptive) {
      prof.t0_ms *= corr[cph];
      prof.slope_ms_per_token *= corr[cph];
      prof.attn_fwd_ms_per_token_ctx *= corr[cph];
      prof.attn_bwd_ms_per_token_ctx *= corr[cph];
      prof.decode_ms_per_row *= corr[cph];
      prof.prefill_ms_per_token *= corr[cph];
    }
    std::vector<int64_t> vtc_admitted;
    if (cfg.vtc && !(temporal && ft_block))
      vtc_admitted = admit_requests_vtc(queue, running, mem, sched, vtc);
    IterationPlan plan, fplan;
    if (spatial) {
      // inference partition: sized so its slowed iteration (x gamma / rho) fits the budget
      FtState idle = ft;
      idle.phase = FtPhase::Idle;
      plan = plan_iteration(queue, running, idle, prof, sched, mem, budget / split.inf_factor());
    } else if (!temporal) {
      plan = plan_iteration(queue, running, ft, prof, sched, mem, budget);
    } else if (ft_block) {
      plan = plan_ft_block(ft, prof, cfg.sched);
    } else {
      FtState idle = ft;  // inference-only iteration
      idle.phase = FtPhase::Idle;
      plan = plan_iteration(queue, running, idle, prof, sched, mem, budget);
      if (plan.c == 0 && ft.L > 0) {  // nothing to serve: the finetuning iteration runs now
        ft_block = true;
        plan = plan_ft_block(ft, prof, cfg.sched);
      }
    }
    // spatial: the tick is the inference iteration slowed by gamma / rho (one budget period when
    // there is no inference work); the finetuning partition gets (1 - rho) / gamma of it
    double tick = 0.0;
    if (spatial) {
      tick = plan.c > 0 ? plan.predicted_ms * split.inf_factor() : budget;
      std::deque<Request> no_q;
      std::vector<Request> no_r;
      SchedulerConfig fs = sched;
      fs.external_admission = true;
      fplan = plan_iteration(no_q, no_r, ft, prof, fs, mem, prof.t0_ms + tick * split.ft_factor());
      if (!enforce_dependencies(fplan, ft)) {
        st.ok = false;
        return st;
      }
    }
    if (!enforce_dependencies(plan, ft)) {
      st.ok = false;
      return st;
    }
    // build the step
    StepInput in;
    for (int i : plan.decode) {
      const Request& r = running[i];
      StepSegment g;
      g.kind = 0;
      g.tokens = {r.last_token};
      g.ctx_start = r.context();
      g.pages = &r.pages;
      g.sample = true;
      in.segs.push_back(std::move(g));
    }
    for (const PrefillChunk& pc : plan.prefill) {
      const Request& r = running[pc.req];
      StepSegment g;
      g.kind = 1;
      for (int t = 0; t < pc.len; ++t) g.tokens.push_back(synth_token(r.id, pc.start + t, cfg.vocab));
      g.ctx_start = pc.start;
      g.pages = &r.pages;
      g.sample = pc.start + pc.len == r.prompt_len;
      in.segs.push_back(std::move(g));
    }
    int64_t s = plan.s;  // (spatial: the finetuning partition's, set after the steps)
    if (s > 0) {
      in.ft_phase = plan.ft_phase;
      in.ft_L = ft.L;
      in.ft_s = (int)s;
      in.ft_pages = &ft_pages;
      if (plan.ft_phase == FtPhase::Forward) {
        in.ft_l = ft.l;
        StepSegment g;
        g.kind = 2;
        g.tokens.assign(ft_tokens.begin() + ft.l, ft_tokens.begin() + ft.l + s);
        g.ctx_start = ft.l;
        g.pages = &ft_pages;
        g.adapter = true;
        in.segs.push_back(std::move(g));
        for (int64_t i = ft.l; i < ft.l + s; ++i)
          in.ft_targets.push_back(i + 1 < ft.L ? ft_tokens[i + 1] : -1);
      } else {
        in.ft_l = plan.bwd[0].lj;
        in.ft_layer = plan.bwd[0].layer;
        in.ft_s = plan.bwd[0].s;
        in.extra_bwd.assign(plan.bwd.begin() + 1, plan.bwd.end());
      }
    }
    StepOutput out;
    if (exec) {
      in.cycle_begin = cycle_t;
      if (!(spatial && in.segs.empty()) && !exec->run(in, out)) {
        st.ok = false;
        return st;
      }
      cycle_t = out.t_end.time_since_epoch().count() ? out.t_end : std::chrono::steady_clock::now();
    } else {
      out.ms = plan.predicted_ms;
      out.device_ms = plan.predicted_ms;
      out.next_tokens.assign(in.segs.size(), 0);
    }
    if (spatial) {
      // the finetuning partition's windows (their kernels run on the engine too; the clock
      // charges the modelled concurrency, not their dedicated-GPU time)
      if (exec && fplan.s > 0) {
        StepInput fi;
        fi.ft_phase = fplan.ft_phase;
        fi.ft_L = ft.L;
        fi.ft_pages = &ft_pages;
        if (fplan.ft_phase == FtPhase::Forward) {
          fi.ft_l = ft.l;
          fi.ft_s = (int)fplan.s;
          StepSegment g;
          g.kind = 2;
          g.tokens.assign(ft_tokens.begin() + ft.l, ft_tokens.begin() + ft.l + fplan.s);
          g.ctx_start = ft.l;
          g.pages = &ft_pages;
          g.adapter = true;
          fi.segs.push_back(std::move(g));
          for (int64_t i = ft.l; i < ft.l + fplan.s; ++i) fi.ft_targets.push_back(i + 1 < ft.L ? ft_tokens[i + 1] : -1);
        } else {
          fi.ft_l = fplan.bwd[0].lj;
          fi.ft_layer = fplan.bwd[0].layer;
          fi.ft_s = fplan.bwd[0].s;
          fi.extra_bwd.assign(fplan.bwd.begin() + 1, fplan.bwd.end());
        }
        StepOutput fo;
        fi.cycle_begin = cycle_t;
        if (!exec->run(fi, fo)) {
          st.ok = false;
          return st;
        }
        cycle_t = fo.t_end.time_since_epoch().count() ? fo.t_end : std::chrono::steady_clock::now();
      }
      // the tick replaces the inference step's own time on the clock (measured x gamma / rho
      // with an executor, predicted otherwise)
      const double t_inf = exec && !cfg.sim_clock && plan.c > 0 ? out.ms : plan.predicted_ms;
      tick = plan.c > 0 ? t_inf * split.inf_factor() : budget;
      out.ms = tick;
      out.device_ms = tick;
      plan.s = s = fplan.s;
      plan.ft_phase = fplan.ft_phase;
      plan.ft_layer = fplan.ft_layer;
      plan.ft_l = fplan.ft_l;
      plan.bwd = fplan.bwd;
      plan.predicted_ms = tick;
    }
    if (cfg.adaptive && !spatial && plan.predicted_ms > 0 && out.device_ms > 0) {
      const int ph = plan.ft_phase == FtPhase::Forward ? 1 : (plan.ft_phase == FtPhase::Backward ? 2 : 0);
      // the step ran with corr[cph]; blend towards the measured ratio of its own phase
      if (use_cal) {
        cal.update(cal.features(plan), out.device_ms);
      } else {
        const double r = corr[cph] * std::max(0.8, std::min(1.25, out.device_ms / plan.predicted_ms));
        corr[ph] = std::max(0.5, std::min(2.0, 0.8 * corr[ph] + 0.2 * r));
      }
      if (cfg.tail_target > 0 && plan.c > 0) {
        const double x = out.device_ms / plan.predicted_ms;
        if (resid.size() < 96) resid.push_back(x);
        else resid[resid_pos++ % 96] = x;
        if (resid.size() >= 12) {
          std::vector<double> srt(resid);
          const size_t k = (size_t)std::ceil(0.95 * (double)srt.size()) - 1;
          std::nth_element(srt.begin(), srt.begin() + k, srt.end());
          const double q95 = std::max(1.0, srt[k]);
          budget = std::max(0.5 * cfg.budget_ms, cfg.tail_target * cfg.sched.tpot_slo_ms / q95);
        }
      }
    }
    if (exec && cfg.sim_clock) out.ms = plan.predicted_ms;
    now += out.ms;
    // advance request state
    int seg = 0;
    for (int i : plan.decode) {
      Request& r = running[i];
      r.last_token = out.next_tokens[seg++];
      r.emitted += 1;
      if (timed) {
        st.gen_tokens += 1;
        // prepopulated requests have no emission time before their first decode in the run
        if (r.last_emit_ms > -1e17 && r.last_emit_ms >= 0.0) st.itl_ms.push_back(now - r.last_emit_ms);
      }
      r.last_emit_ms = now;
      if (r.done()) r.completion_ms = now;
    }
    for (const PrefillChunk& pc : plan.prefill) {
      Request& r = running[pc.req];
      r.prefilled += pc.len;
      if (!r.in_prefill()) {
        r.last_token = out.next_tokens[seg];
        r.emitted = 1;
        r.first_token_ms = now;
        r.last_emit_ms = now;
        if (timed) st.gen_tokens += 1;
        if (r.done()) r.completion_ms = now;
      }
      ++seg;
    }
    if (cfg.vtc) {  // generated tokens w_q (decodes + prefill-completing first tokens), FT w_r
      for (int i : plan.decode) vtc.charge(running[i].tenant, vtc.w_q);
      for (const PrefillChunk& pc : plan.prefill)
        if (!running[pc.req].in_prefill()) vtc.charge(running[pc.req].tenant, vtc.w_q);
      if (cfg.ft_tenant >= 0 && s > 0) vtc.charge(cfg.ft_tenant, vtc.w_r * (double)s);
      st.vtc_spread_max = std::max(st.vtc_spread_max, vtc.queued_spread());
      const bool both = vtc.queued.size() > 1 && vtc.queued[0] > 0 && vtc.queued[1] > 0;
      const double dW = vtc.service.size() > 1 ? vtc.service[0] - vtc.service[1] : 0.0;
      if (both) {
        if (!pair_on) pair_on = true, pair_lo = pair_hi = dW;
        pair_lo = std::min(pair_lo, dW);
        pair_hi = std::max(pair_hi, dW);
        st.vtc_pair_gap_max = std::max(st.vtc_pair_gap_max, pair_hi - pair_lo);
      } else {
        pair_on = false;
      }
    }
    // retire finished requests
    int64_t completed = 0;
    for (size_t i = 0; i < running.size();) {
      Request& r = running[i];
      if (r.done()) {
        ++completed;
        if (r.arrival_ms > -1e17) {
          const double ttft = r.first_token_ms - r.arrival_ms;
          const double tpot = r.gen_len > 1 ? (r.completion_ms - r.first_token_ms) / (r.gen_len - 1) : 0.0;
          st.ttft_ms.push_back(ttft);
          st.tpot_ms.push_back(tpot);
          st.requests_done += 1;
          if (tpot <= cfg.sched.tpot_slo_ms && ttft <= cfg.sched.ttft_slo_ms) st.requests_slo_ok += 1;
          if (r.arrival_ms >= timed_t0) {
            st.timed_done += 1;
            if (tpot <= cfg.sched.tpot_slo_ms && ttft <= cfg.sched.ttft_slo_ms) st.timed_slo_ok += 1;
          }
          if ((int)st.tenant_done.size() <= r.tenant) st.tenant_done.resize(r.tenant + 1, 0);
          st.tenant_done[r.tenant] += 1;
        }
        mem.release(r.pages);
        running.erase(running.begin() + i);
      } else {
        ++i;
      }
    }
    // finetuning progress
    const FtPhase ph = ft.phase;
    if (plan.ft_phase == FtPhase::Backward) {
      for (const BwdWindow& bw : plan.bwd) advance_finetune(ft, bw.s);
    } else {
      advance_finetune(ft, s);
    }
    if (timed) {
      if (ph == FtPhase::Forward) {
        st.ft_fwd_tokens += s;
        st.ft_fwd_ms += out.device_ms;
      } else if (ph == FtPhase::Backward) {
        st.ft_bwd_tokens += s;
        st.ft_bwd_ms += out.device_ms;
      }
      st.inf_tokens += plan.c;
      st.timed_ms += out.ms;
      st.timed_device_ms += out.device_ms;
    }
    // temporal sharing: count inference-only iterations, decide the next finetuning one
    if (temporal && !ft_block && ft.L > 0) {
      ++inf_since_ft;
      if (cfg.policy == Policy::TemporalFixed) {
        ft_block = inf_since_ft >= std::max(1, cfg.temporal_n);
      } else {
        ft_block = dts_step(dts, (double)queue.size(),
                            (double)(plan.decode.size() + plan.prefill.size()), (double)arrived,
                            (double)completed);
      }
    }
    if (ft.phase == FtPhase::Done) {
      ft_block = false;
      inf_since_ft = 0;
      if (exec && !exec->adam()) {
        st.ok = false;
        return st;
      }
      if (timed) st.minibatches_done += 1;
      ft.phase = FtPhase::Forward;
      ft.minibatch += 1;
      ft.l = 0;
      ft.layer = 0;
      ft.lj = 0;
      for (int i = 0; i < ft.L; ++i) ft_tokens[i] = synth_token(-1 - ft.minibatch, i, cfg.vocab);
    }
    IterLog lg;
    lg.t_ms = now;
    lg.pred_ms = plan.predicted_ms;
    lg.ms = out.ms;
    lg.device_ms = out.device_ms;
    lg.c = (int)plan.c;
    lg.s = (int)s;
    lg.phase = (int)plan.ft_phase;
    lg.layer = plan.ft_layer;
    lg.l = plan.ft_l;
    lg.n_decode = (int)plan.decode.size();
    lg.n_prefill = (int)plan.prefill.size();
    lg.n_running = (int)running.size();
    lg.n_queue = (int)queue.size();
    lg.timed = timed;
    st.log.push_back(lg);
    st.iters += 1;
  }
  // timed-region arrivals still queued or prefilling whose first-token wait already breaks
  // the TTFT SLO are misses; in-flight ones that have their first token count once done
  auto unfinished_miss = [&](const Request& r) {
    return r.arrival_ms >= timed_t0 && r.arrival_ms > -1e17 && r.first_token_ms < 0 &&
           now - r.arrival_ms > cfg.sched.ttft_slo_ms;
  };
  for (const Request& r : queue) st.timed_unfinished_miss += unfinished_miss(r) ? 1 : 0;
  for (const Request& r : running) st.timed_unfinished_miss += unfinished_miss(r) ? 1 : 0;
  st.tenant_service = vtc.service;
  return st;
}

}  // namespace coserve
