// tests/cpp/test_host.cpp -- native unit tests of the host C++ runtime (include/coserve/),
// the SPEC.md worked examples for the modules the reference left as spec only
// (cost_model SPEC.md:353-379, coserve_scheduler :421-447, workload_gen :635-652).
// Built and run by tests/test_host_cpp.py (g++, no GPU).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <limits>
#include <string>
#include <vector>

#include "coserve/coserve_loop.hpp"
#include "coserve/cost_model.hpp"
#include "coserve/scheduler.hpp"
#include "coserve/vtc.hpp"
#include "coserve/workload.hpp"

using namespace coserve;

static int failures = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    if (!(cond)) {                                                             \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);              \
      ++failures;                                                              \
    }                                                                          \
  } while (0)

static bool near(double a, double b, double tol = 1e-9) { return std::fabs(a - b) <= tol; }

static void test_cost_model() {
  LatencyProfile p;
  p.t0_ms = 2;
  p.slope_ms_per_token = 0.01;
  p.knee_tokens = 4096;
  CHECK(near(latency(p, 0, 0), 2.0));                        // f(0,0) = t0
  CHECK(near(latency(p, 1000, 0), 12.0));
  CHECK(near(latency(p, 4096 + 100, 0), 44.96));
  LatencyProfile q = p;
  q.knee_tokens = std::numeric_limits<double>::infinity();
  CHECK(max_finetune_tokens(q, 1000, 50.0) == 3800);
  CHECK(max_finetune_tokens(q, 1000, latency(q, 1000, 7)) == 7);  // SPEC.md:370 inclusive
  CHECK(max_finetune_tokens(q, 10000, 50.0) == 0);          // f(c,0) > budget
  for (int c : {0, 17, 1000, 3000})
    for (double b : {5.0, 20.0, 50.0, 77.7}) {
      const int64_t s = max_finetune_tokens(p, c, b);
      if (s > 0) CHECK(latency(p, c, s) <= b);
      if (latency(p, c, 0) <= b) CHECK(latency(p, c, s + 1) > b);  // exact argmax
    }
  bool threw = false;
  try {
    latency(p, -1, 0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

static void test_memory_model() {
  MemoryModel empty(8, 16);
  std::vector<int32_t> pg;
  CHECK(empty.try_admit(1, &pg) && pg.size() == 1);
  MemoryModel m(3, 16);
  CHECK(!m.try_admit(60, &pg));                              // SPEC.md:378 needs 4
  CHECK(m.free_pages() == 3);                                // atomic: nothing reserved
  MemoryModel full(2, 16);
  CHECK(full.try_admit(32, &pg));
  CHECK(!full.try_admit(1, &pg));                            // full pool
}

static void test_advance_finetune() {
  FtState ft;
  ft.L = 8;
  ft.n_layers = 2;
  ft.phase = FtPhase::Forward;
  std::vector<int> trace;
  for (int s : {3, 3, 2}) {
    advance_finetune(ft, s);
    trace.push_back(ft.l);
  }
  CHECK(trace == std::vector<int>({3, 6, 8}));
  CHECK(ft.phase == FtPhase::Backward && ft.layer == 1 && ft.lj == 8);
  FtState b;
  b.L = 4;
  b.n_layers = 2;
  b.phase = FtPhase::Forward;
  advance_finetune(b, 4);
  int iters = 0;
  while (b.phase == FtPhase::Backward) {
    advance_finetune(b, 4);
    ++iters;
  }
  CHECK(iters == 2 && b.phase == FtPhase::Done);
  FtState z = ft;
  advance_finetune(z, 0);
  CHECK(z.lj == ft.lj && z.layer == ft.layer);               // s = 0 -> unchanged
  advance_finetune(z, 100);                                   // clipped, never an error
  CHECK(z.layer == 0 && z.lj == 8);
}

static void test_plan_iteration() {
  LatencyProfile p;
  p.t0_ms = 0;
  p.slope_ms_per_token = 1.0;  // budget 600 ms -> 600 tokens
  SchedulerConfig cfg;
  cfg.chunk_size = 512;
  MemoryModel mem(1000, 16);
  std::deque<Request> q;
  std::vector<Request> running;
  for (int i = 0; i < 3; ++i) {
    Request r;
    r.id = i;
    r.prompt_len = 10;
    r.gen_len = 100;
    r.prefilled = 10;
    r.emitted = 1;
    running.push_back(r);
  }
  Request big;
  big.id = 3;
  big.prompt_len = 1024;
  big.gen_len = 10;
  q.push_back(big);
  FtState ft;
  ft.L = 4096;
  ft.n_layers = 2;
  ft.phase = FtPhase::Forward;
  ft.minibatch = 0;
  IterationPlan pl = plan_iteration(q, running, ft, p, cfg, mem, 600.0);
  CHECK(pl.decode.size() == 3);
  CHECK(pl.prefill.size() == 1 && pl.prefill[0].len == 512);
  CHECK(pl.c == 515 && pl.s == 85);
  CHECK(enforce_dependencies(pl, ft));
  // no inference work: c = 0, s = max under budget (work conservation)
  std::deque<Request> q2;
  std::vector<Request> r2;
  IterationPlan p2 = plan_iteration(q2, r2, ft, p, cfg, mem, 600.0);
  CHECK(p2.c == 0 && p2.s == 600);
  // c consumes the whole budget -> s = 0
  std::vector<Request> r3;
  for (int i = 0; i < 64; ++i) {
    Request r;
    r.id = 100 + i;
    r.prompt_len = 1;
    r.gen_len = 50;
    r.prefilled = 1;
    r.emitted = 1;
    r3.push_back(r);
  }
  IterationPlan p3 = plan_iteration(q2, r3, ft, p, cfg, mem, 60.0);
  CHECK(p3.c == 60 && p3.s == 0);
  // dependencies
  FtState fwd = ft;
  fwd.l = 5;
  IterationPlan bad;
  bad.s = 4;
  bad.ft_phase = FtPhase::Backward;
  bad.ft_minibatch = 0;
  CHECK(!enforce_dependencies(bad, fwd));
  FtState bwd = ft;
  bwd.l = bwd.L;
  bwd.phase = FtPhase::Backward;
  bwd.layer = 1;
  CHECK(enforce_dependencies(bad, bwd));
  IterationPlan mixed = bad;
  mixed.ft_minibatch = 1;
  CHECK(!enforce_dependencies(mixed, bwd));
}

// with per-row inference slopes steeper than the common FT slope, the inference rows
// alone must still fit the budget (the planner sizes them with inference_cost), and a
// single-profile backward window is capped at the engine's max_tokens
static void test_plan_row_slopes_and_caps() {
  LatencyProfile p;
  p.t0_ms = 1.0;
  p.slope_ms_per_token = 0.01;
  p.decode_ms_per_row = 0.05;       // 5x the common slope
  p.prefill_ms_per_token = 0.03;
  SchedulerConfig cfg;
  cfg.chunk_size = 512;
  cfg.max_tokens = 4096;
  MemoryModel mem(4000, 16);
  std::deque<Request> q;
  std::vector<Request> running;
  for (int i = 0; i < 300; ++i) {
    Request r;
    r.id = i;
    r.prompt_len = 10;
    r.gen_len = 100;
    r.prefilled = i < 250 ? 10 : 0;  // 250 decoding, 50 in prefill
    r.emitted = i < 250 ? 1 : 0;
    running.push_back(r);
  }
  FtState ft;
  ft.L = 8192;
  ft.n_layers = 2;
  ft.phase = FtPhase::Forward;
  ft.minibatch = 0;
  const double budget = 10.0;
  IterationPlan pl = plan_iteration(q, running, ft, p, cfg, mem, budget);
  int64_t n_pre = 0;
  for (const auto& c : pl.prefill) n_pre += c.len;
  CHECK(inference_cost(p, (int64_t)pl.decode.size(), n_pre) <= budget);
  CHECK(pl.decode.size() == 180);   // (10 - 1) / 0.05
  CHECK(pl.predicted_ms <= budget + 1e-9);
  // single-profile backward window: capped by max_tokens even with a larger window cap
  LatencyProfile flat;
  flat.t0_ms = 0;
  flat.slope_ms_per_token = 1e-4;
  SchedulerConfig c2;
  c2.max_tokens = 1024;
  c2.max_ft_window = 8192;
  FtState b;
  b.L = 8192;
  b.n_layers = 2;
  b.l = b.L;
  b.phase = FtPhase::Backward;
  b.layer = 1;
  b.lj = 8192;
  b.minibatch = 0;
  std::deque<Request> q2;
  std::vector<Request> r2;
  IterationPlan pb = plan_iteration(q2, r2, b, flat, c2, mem, 50.0);
  CHECK(pb.s == 1024 && pb.bwd.size() == 1 && pb.bwd[0].s == 1024);
}

static void test_workload() {
  WorkloadConfig w;
  w.rate_rps = 0;
  CHECK(generate_trace(w, 1).empty());
  w.rate_rps = 4;
  w.duration_s = 1200;
  auto t = generate_trace(w, 3);
  CHECK(std::fabs((double)t.size() - 4800.0) <= 208.0);      // SPEC.md:642 (+-3 sigma)
  auto t2 = generate_trace(w, 3);
  bool same = t.size() == t2.size();
  for (size_t i = 0; same && i < t.size(); ++i)
    same = t[i].time_ms == t2[i].time_ms && t[i].prompt_len == t2[i].prompt_len;
  CHECK(same);                                               // determinism
  for (size_t i = 1; i < t.size(); ++i) CHECK(t[i].time_ms >= t[i - 1].time_ms);
  for (auto& a : t) CHECK(a.prompt_len >= 16 && a.prompt_len <= 4096 && a.gen_len >= 8 && a.gen_len <= 1024);
  auto r = rescale(t, 2.0);
  CHECK(near(r.back().time_ms * 2.0, t.back().time_ms, 1e-6));
  bool threw = false;
  try {
    rescale(t, 0.0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  w.burst_amplitude = 1.5;
  threw = false;
  try {
    generate_trace(w, 1);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

static void test_sim_loop() {
  // one request, prompt 10, gen 5, 10 ms/iteration -> TTFT 10, TPOT 10
  LoopConfig c;
  c.prof.t0_ms = 10;
  c.prof.slope_ms_per_token = 0;
  c.budget_ms = 50;
  c.ft_seq_len = 0;
  c.timed_iters = 10;
  c.workload.rate_rps = 0;  // no random arrivals; inject manually below via prepopulate = 0
  LoopStats st = run_coserve(c, nullptr);
  CHECK(st.ok && st.requests_done == 0);                     // empty trace -> zero metrics
  // token accounting: a finished mini-batch processes L forward + N*L backward tokens
  LoopConfig f;
  f.prof.t0_ms = 1;
  f.prof.slope_ms_per_token = 0.01;
  f.budget_ms = 50;
  f.ft_seq_len = 64;
  f.n_layers = 3;
  f.timed_iters = 40;
  f.workload.rate_rps = 0;
  LoopStats fs = run_coserve(f, nullptr);
  CHECK(fs.ok && fs.minibatches_done >= 1);
  CHECK(fs.ft_fwd_tokens >= 64 * fs.minibatches_done);
  CHECK(fs.ft_bwd_tokens >= 3 * 64 * fs.minibatches_done);
  // SLO safety: predicted latency <= budget whenever inference is active
  LoopConfig h;
  h.prof.t0_ms = 5;
  h.prof.slope_ms_per_token = 0.01;
  h.budget_ms = 50;
  h.ft_seq_len = 2048;
  h.n_layers = 8;
  h.timed_iters = 400;
  h.workload.rate_rps = 20;
  h.total_pages = 1 << 14;
  LoopStats hs = run_coserve(h, nullptr);
  CHECK(hs.ok);
  for (auto& lg : hs.log)
    if (lg.c > 0) CHECK(lg.pred_ms <= 50.0 + 1e-9);
}

// SPEC.md fairness_vtc examples (Appendix C)
static void test_vtc() {
  VtcLedger v;  // sole tenant rejoining an empty system after tenant l left with c_l = 500
  v.ensure(1);
  v.counter[1] = 100.0;
  v.c_last = 500.0;
  v.on_arrival(1);
  CHECK(near(v.counter[1], 500.0));
  VtcLedger a;  // active tenants {200, 300}, rejoiner at 50 -> lifted to 200
  a.ensure(2);
  a.counter = {200.0, 300.0, 50.0};
  a.queued = {1, 1, 0};
  a.on_arrival(2);
  CHECK(near(a.counter[2], 200.0));
  a.counter[2] = 250.0;  // already queued -> no lift
  a.on_arrival(2);
  CHECK(near(a.counter[2], 250.0) && a.queued[2] == 2);
  VtcLedger s;  // select: counters {A:10, B:5} -> B ; tie 7 vs 7 -> lowest id
  s.ensure(1);
  s.counter = {10.0, 5.0};
  std::deque<Request> q(2);
  q[0].tenant = 0;
  q[1].tenant = 1;
  CHECK(s.select(q) == 1);
  s.counter = {7.0, 7.0};
  CHECK(s.select(q) == 0);
  VtcLedger c;  // charges: w_p = 1 prompt 100 -> +100 ; w_q = 2, 5 tokens -> +10 ; w_r = 0.5 x 64 -> +32
  c.w_r = 0.5;
  c.ensure(0);
  c.queued[0] = 1;
  c.on_admit(0, 100);
  CHECK(near(c.counter[0], 100.0) && near(c.c_last, 100.0));
  c.charge(0, c.w_q * 5);
  CHECK(near(c.counter[0], 110.0));
  c.charge(0, c.w_r * 64);
  CHECK(near(c.counter[0], 142.0) && near(c.service[0], 142.0));
}

// online calibration (coserve/calibrate.hpp): a "true" box whose coefficients differ from the
// profiled prior by up to +-20% each; after ~400 measured iterations of mixed plans the
// calibrated model predicts fresh plans within 2% (the prior is off by up to ~15%), the
// prediction equals the planner's own predicted_ms for ctx-term profiles, and coefficients
// stay inside [1/2, 2] x prior under adversarial measurements
static void test_calibrator() {
  LatencyProfile prior;
  prior.t0_ms = 4.8;
  prior.slope_ms_per_token = 0.013;
  prior.bwd_token_weight = 0.026;
  prior.attn_fwd_ms_per_token_ctx = 7.1e-7;
  prior.attn_bwd_ms_per_token_ctx = 5.5e-8;
  prior.bwd_layer0_weight = 0.25;
  prior.decode_ms_per_row = 0.007;
  prior.prefill_ms_per_token = 0.0099;
  prior.fwd_window_ms = 2.3;
  CHECK(CostCalibrator::applicable(prior));
  CHECK(!CostCalibrator::applicable(LatencyProfile{}));
  LatencyProfile truth = prior;
  truth.t0_ms *= 1.12;
  truth.decode_ms_per_row *= 0.85;
  truth.prefill_ms_per_token *= 1.1;
  truth.fwd_window_ms *= 0.8;
  truth.slope_ms_per_token *= 0.92;
  truth.attn_fwd_ms_per_token_ctx *= 1.2;
  truth.bwd_token_weight *= 1.15 / 0.92;  // backward token cost x 1.15
  truth.attn_bwd_ms_per_token_ctx *= 0.85;
  CostCalibrator cal(prior), truth_model(truth);
  TraceRng rng(11);
  auto random_plan = [&](int kind) {
    IterationPlan p;
    const int nd = 40 + (int)(rng.uniform() * 60), np = rng.uniform() < 0.5 ? 0 : 512;
    p.decode.resize(nd);
    p.c = nd + np;
    if (kind == 1) {
      p.ft_phase = FtPhase::Forward;
      p.s = 200 + (int64_t)(rng.uniform() * 1800);
      p.ft_l = (int)(rng.uniform() * 6000);
    } else if (kind == 2) {
      p.ft_phase = FtPhase::Backward;
      int lj = 8192, layer = 31 - (int)(rng.uniform() * 31);
      for (int w = 0; w < 4 && layer >= 0; ++w) {
        const int s = std::min(lj, 1024 + (int)(rng.uniform() * 7168));
        p.bwd.push_back(BwdWindow{layer, lj, s});
        p.s += s;
        lj -= s;
        if (lj == 0) { layer -= 1; lj = 8192; }
      }
      p.ft_layer = p.bwd[0].layer;
      p.ft_l = p.bwd[0].lj;
    }
    return p;
  };
  for (int it = 0; it < 400; ++it) {
    const IterationPlan p = random_plan(it % 3);
    const double y = truth_model.predict(truth_model.features(p)) * (1.0 + 0.02 * (rng.uniform() - 0.5));
    cal.update(cal.features(p), y);
  }
  CostCalibrator prior_model(prior);
  double worst = 0, worst_prior = 0;
  for (int it = 0; it < 300; ++it) {
    const IterationPlan p = random_plan(it % 3);
    const double y = truth_model.predict(truth_model.features(p));
    worst = std::max(worst, std::fabs(cal.predict(cal.features(p)) / y - 1.0));
    worst_prior = std::max(worst_prior, std::fabs(prior_model.predict(prior_model.features(p)) / y - 1.0));
  }
  CHECK(worst < 0.02);
  CHECK(worst_prior > 0.08);
  // the calibrated profile drives the planner's cost functions to the same prediction
  {
    const LatencyProfile q = cal.profile();
    const IterationPlan f = random_plan(1), b = random_plan(2);
    const double pf = inference_cost(q, (int64_t)f.decode.size(), f.c - (int64_t)f.decode.size()) +
                      ft_fwd_cost(q, f.ft_l, f.s);
    double pb = inference_cost(q, (int64_t)b.decode.size(), b.c - (int64_t)b.decode.size());
    for (const BwdWindow& w : b.bwd) pb += ft_bwd_cost(q, w.lj, w.s, w.layer);
    CHECK(std::fabs(pf / cal.predict(cal.features(f)) - 1.0) < 1e-9);
    CHECK(std::fabs(pb / cal.predict(cal.features(b)) - 1.0) < 1e-9);
  }
  // adversarial measurements (10x) cannot push a coefficient past 2x its prior
  CostCalibrator bad(prior);
  for (int it = 0; it < 200; ++it) {
    const IterationPlan p = random_plan(it % 3);
    bad.update(bad.features(p), 10.0 * prior_model.predict(prior_model.features(p)));
  }
  CostCalibrator ref(prior);
  for (int i = 0; i < CostCalibrator::K; ++i) CHECK(bad.theta()[i] <= 2.0 * ref.theta()[i] + 1e-15);
}

int main() {
  test_cost_model();
  test_memory_model();
  test_advance_finetune();
  test_plan_iteration();
  test_plan_row_slopes_and_caps();
  test_workload();
  test_sim_loop();
  test_vtc();
  test_calibrator();
  if (failures) {
    std::printf("%d failure(s)\n", failures);
    return 1;
  }
  std::printf("all host tests passed\n");
  return 0;
}
