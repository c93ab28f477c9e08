// coserve_run.cpp -- cs_coserve_run: the C++ co-serving loop (include/coserve/coserve_loop.hpp)
// driving the GPU engine through its own C ABI (cs_step / cs_adam_step), or a simulated clock.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "coserve/coserve_loop.hpp"
#include "coserve_cuda.h"

namespace cs {
int set_error(int code, const std::string& msg);
}

namespace {

class GpuExecutor : public coserve::StepExecutor {
 public:
  explicit GpuExecutor(cs_engine* e) : e_(e) {}
  int64_t h2d = 0, d2h = 0;
  bool count = false;
  bool run(const coserve::StepInput& in, coserve::StepOutput& out) override {
    tokens_.clear();
    segs_.clear();
    pt_.clear();
    int row = 0;
    for (const auto& g : in.segs) {
      cs_segment s{};
      s.kind = g.kind;
      s.q_start = row;
      s.q_len = (int)g.tokens.size();
      s.ctx_start = g.ctx_start;
      s.page_off = (int)pt_.size();
      const int need = (g.ctx_start + s.q_len + page_size_ - 1) / page_size_;
      s.n_pages = std::min<int>(need, (int)g.pages->size());
      pt_.insert(pt_.end(), g.pages->begin(), g.pages->begin() + s.n_pages);
      s.sample = g.sample ? 1 : 0;
      s.adapter = g.adapter ? 1 : 0;
      tokens_.insert(tokens_.end(), g.tokens.begin(), g.tokens.end());
      segs_.push_back(s);
      row += s.q_len;
    }
    cs_iteration_plan p{};
    p.n_tokens = row;
    p.tokens = tokens_.data();
    p.n_segments = (int)segs_.size();
    p.segments = segs_.data();
    cs_ft_window& w = p.ft;
    w.phase = (int)in.ft_phase == 1 ? CS_FT_FORWARD : ((int)in.ft_phase == 2 ? CS_FT_BACKWARD : CS_FT_NONE);
    if (w.phase != CS_FT_NONE) {
      w.seq_len = in.ft_L;
      w.l = in.ft_l;
      w.s = in.ft_s;
      w.layer = in.ft_layer;
      w.targets = in.ft_targets.empty() ? nullptr : in.ft_targets.data();
      w.page_off = (int)pt_.size();
      w.n_pages = (int)in.ft_pages->size();
      pt_.insert(pt_.end(), in.ft_pages->begin(), in.ft_pages->end());
    }
    extra_.clear();
    for (const auto& b : in.extra_bwd) {
      cs_ft_window x = w;
      x.l = b.lj;
      x.s = b.s;
      x.layer = b.layer;
      x.targets = nullptr;
      extra_.push_back(x);
    }
    p.n_extra_bwd = (int)extra_.size();
    p.extra_bwd = extra_.empty() ? nullptr : extra_.data();
    p.page_table = pt_.data();
    p.page_table_len = (int)pt_.size();
    next_.assign(std::max<size_t>(1, segs_.size()), -1);
    cs_step_result r{};
    r.next_tokens = next_.data();
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = cs_step(e_, &p, &r);
    const auto t1 = std::chrono::steady_clock::now();
    if (rc != CS_OK) return false;
    if (count) {
      h2d += (int64_t)(tokens_.size() + pt_.size() + in.ft_targets.size()) * 4 +
             (int64_t)segs_.size() * (int64_t)sizeof(cs_segment);
      int ns = 0;
      for (const auto& g : in.segs) ns += g.sample ? 1 : 0;
      d2h += (int64_t)ns * 4 + (w.phase == CS_FT_FORWARD ? (int64_t)in.ft_s * 4 : 0);
    }
    out.next_tokens.assign(next_.begin(), next_.begin() + in.segs.size());
    // the clock advances by the whole cycle since the previous step returned (the loop's
    // planning and bookkeeping, the Adam step, this step's enqueue, execution and sync)
    const auto tb = in.cycle_begin.time_since_epoch().count() ? in.cycle_begin : t0;
    out.ms = std::chrono::duration<double, std::milli>(t1 - tb).count();
    out.t_end = t1;
    out.device_ms = r.iteration_ms;
    // TP group: one loop per rank -> the clock must be rank-invariant (max over ranks), so
    // every rank admits, plans and corrects identically
    double clk[2] = {out.ms, out.device_ms};
    if (cs_engine_tp_sync_max(e_, clk, 2) != CS_OK) return false;
    out.ms = clk[0];
    out.device_ms = clk[1];
    return true;
  }
  bool adam() override { return cs_adam_step(e_, 1e-4f, 0.9f, 0.999f, 1e-8f) == CS_OK; }
  int page_size_ = 16;

 private:
  cs_engine* e_;
  std::vector<int32_t> tokens_, pt_, next_;
  std::vector<cs_segment> segs_;
  std::vector<cs_ft_window> extra_;
};

double pct(std::vector<double> v, double q) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const size_t i = std::min(v.size() - 1, (size_t)std::ceil(q * v.size()) - (q > 0 ? 1 : 0));
  return v[i];
}

}  // namespace

// engine.cu accessors
extern "C" int cs_engine_pool_info(cs_engine* e, int32_t* n_layers, int32_t* vocab,
                                   int32_t* page_size, int64_t* n_pages);

extern "C" int cs_coserve_run(cs_engine* e, const cs_coserve_config* c, cs_coserve_stats* stats,
                              cs_iter_log* log, int64_t log_cap, int64_t* log_len) {
  if (!c || !stats) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_coserve_run: null argument");
  coserve::LoopConfig L;
  L.sched.max_batch = c->max_batch;
  L.sched.chunk_size = c->chunk_size;
  L.sched.tpot_slo_ms = c->tpot_slo_ms;
  L.sched.ttft_slo_ms = c->ttft_slo_ms;
  L.sched.max_tokens = c->max_tokens;
  L.sched.max_ft_window = c->max_ft_window;
  L.prof.t0_ms = c->profile.t0_ms;
  L.prof.slope_ms_per_token = c->profile.slope_ms_per_token;
  L.prof.knee_tokens = c->profile.knee_tokens > 0 ? c->profile.knee_tokens
                                                  : std::numeric_limits<double>::infinity();
  L.prof.bwd_token_weight = c->profile.bwd_token_weight > 0 ? c->profile.bwd_token_weight : 1.0;
  L.prof.attn_fwd_ms_per_token_ctx = c->profile.attn_fwd_ms_per_token_ctx;
  L.prof.attn_bwd_ms_per_token_ctx = c->profile.attn_bwd_ms_per_token_ctx;
  L.prof.bwd_layer0_weight = c->profile.bwd_layer0_weight > 0 ? c->profile.bwd_layer0_weight : 1.0;
  L.prof.decode_ms_per_row = c->profile.decode_ms_per_row > 0 ? c->profile.decode_ms_per_row : 0.0;
  L.prof.prefill_ms_per_token = c->profile.prefill_ms_per_token > 0 ? c->profile.prefill_ms_per_token : 0.0;
  L.prof.fwd_window_ms = c->profile.fwd_window_ms > 0 ? c->profile.fwd_window_ms : 0.0;
  L.sched.multi_layer_bwd = c->multi_layer_bwd != 0;
  L.budget_ms = c->budget_ms > 0 ? c->budget_ms : c->tpot_slo_ms;
  L.growth_tokens = c->growth_tokens;
  L.ft_seq_len = c->ft_seq_len;
  L.warmup_iters = c->warmup_iters;
  L.timed_iters = c->timed_iters;
  L.prepopulate = c->prepopulate;
  L.adaptive = c->adaptive != 0;
  L.calibrate = c->adaptive == 2;  // adaptive 2: per-coefficient online calibration
  L.seed = c->seed;
  if (c->policy < 0 || c->policy > 4)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_coserve_run: policy must be in 0..4");
  L.policy = (coserve::Policy)c->policy;
  if (L.policy == coserve::Policy::Spatial || L.policy == coserve::Policy::Isolate) {
    if (!(c->spatial_rho > 0.0 && c->spatial_rho < 1.0))
      return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_coserve_run: spatial_rho must be in (0, 1)");
    L.split.rho = c->spatial_rho;
    L.split.gamma = c->spatial_gamma >= 1.0 ? c->spatial_gamma : 1.15;
  }
  L.temporal_n = c->temporal_n > 0 ? c->temporal_n : 128;
  L.sim_clock = c->sim_clock != 0;
  L.tail_target = c->tail_target > 0 && c->tail_target <= 1.0 ? c->tail_target : 0.0;
  L.vtc = c->vtc != 0;
  if (L.vtc) {
    L.vtc_wp = c->vtc_wp > 0 ? c->vtc_wp : 1.0;
    L.vtc_wq = c->vtc_wq > 0 ? c->vtc_wq : 2.0;
    L.vtc_wr = c->vtc_wr > 0 ? c->vtc_wr : 1.0;
    L.ft_tenant = c->ft_tenant;
  }
  L.workload.n_tenants = std::max(1, std::min(8, (int)c->n_tenants));
  L.workload.tenant0_share = c->tenant0_share > 0 ? c->tenant0_share : 0.5;
  L.workload.rate_rps = c->rate_rps;
  L.workload.duration_s = c->duration_s;
  L.workload.burst_amplitude = c->burst_amplitude;
  L.workload.burst_period_s = c->burst_period_s > 0 ? c->burst_period_s : 60.0;
  if (c->max_batch < 1 || c->chunk_size < 1 || c->max_tokens < 1 || c->timed_iters < 0 ||
      c->warmup_iters < 0 || c->ft_seq_len < 0)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_coserve_run: bad configuration");
  GpuExecutor* ex = nullptr;
  if (e) {
    int32_t nl, V, P;
    int64_t np;
    cs_engine_pool_info(e, &nl, &V, &P, &np);
    L.n_layers = nl;
    L.vocab = V;
    L.page_size = P;
    L.total_pages = np;
    ex = new GpuExecutor(e);
    ex->page_size_ = P;
  } else {
    L.n_layers = c->n_layers;
    L.vocab = c->vocab;
    L.page_size = c->page_size;
    L.total_pages = c->total_pages;
  }
  // count launches / bytes in the timed region only: run warmup first by splitting the loop
  // is not possible with one trace, so the executor counts from the first timed iteration
  struct Counting : public coserve::StepExecutor {
    GpuExecutor* g;
    int warm;
    bool profile = false;
    int n = 0;
    int64_t launches0 = 0;
    cs_engine* e;
    bool run(const coserve::StepInput& in, coserve::StepOutput& out) override {
      if (n == warm) {
        g->count = true;
        if (profile) cs_engine_set_profiling(e, 1);
        launches0 = cs_engine_launch_count(e);
      }
      ++n;
      return g->run(in, out);
    }
    bool adam() override { return g->adam(); }
  } counting;
  counting.g = ex;
  counting.warm = L.warmup_iters;
  counting.profile = c->profile_timed != 0;
  if (e) cs_engine_reset_ft(e);
  counting.e = e;
  coserve::LoopStats st = coserve::run_coserve(L, ex ? (coserve::StepExecutor*)&counting : nullptr);
  int rc = CS_OK;
  if (!st.ok) rc = cs::set_error(CS_ERR_RUNTIME, std::string("cs_coserve_run failed: ") + cs_last_error());
  *stats = cs_coserve_stats{};
  stats->iters = st.iters;
  stats->timed_ms = st.timed_ms;
  stats->timed_device_ms = st.timed_device_ms;
  stats->ft_fwd_tokens = st.ft_fwd_tokens;
  stats->ft_bwd_tokens = st.ft_bwd_tokens;
  stats->ft_fwd_ms = st.ft_fwd_ms;
  stats->ft_bwd_ms = st.ft_bwd_ms;
  stats->minibatches_done = st.minibatches_done;
  stats->inf_tokens = st.inf_tokens;
  stats->gen_tokens = st.gen_tokens;
  stats->requests_done = st.requests_done;
  stats->requests_slo_ok = st.requests_slo_ok;
  stats->evictions = st.evictions;
  stats->ttft_p50_ms = pct(st.ttft_ms, 0.5);
  stats->ttft_p99_ms = pct(st.ttft_ms, 0.99);
  stats->tpot_p50_ms = pct(st.tpot_ms, 0.5);
  stats->tpot_p99_ms = pct(st.tpot_ms, 0.99);
  std::vector<double> its;
  for (const auto& lg : st.log)
    if (lg.timed && lg.c > 0) its.push_back(lg.ms);
  stats->iter_p50_ms = pct(its, 0.5);
  stats->iter_p99_ms = pct(its, 0.99);
  stats->iter_max_ms = its.empty() ? 0.0 : *std::max_element(its.begin(), its.end());
  for (int t = 0; t < 8; ++t) {
    stats->tenant_service[t] = t < (int)st.tenant_service.size() ? st.tenant_service[t] : 0.0;
    stats->tenant_done[t] = t < (int)st.tenant_done.size() ? st.tenant_done[t] : 0;
  }
  stats->vtc_spread_max = st.vtc_spread_max;
  stats->vtc_pair_gap_max = st.vtc_pair_gap_max;
  stats->itl_p50_ms = pct(st.itl_ms, 0.5);
  stats->itl_p99_ms = pct(st.itl_ms, 0.99);
  stats->itl_max_ms = st.itl_ms.empty() ? 0.0 : *std::max_element(st.itl_ms.begin(), st.itl_ms.end());
  stats->itl_samples = (int64_t)st.itl_ms.size();
  stats->timed_arrivals = st.timed_arrivals;
  stats->timed_done = st.timed_done;
  stats->timed_slo_ok = st.timed_slo_ok;
  stats->timed_unfinished_miss = st.timed_unfinished_miss;
  if (ex) {
    stats->gpu_launches = cs_engine_launch_count(e) - counting.launches0;
    stats->h2d_bytes = ex->h2d;
    stats->d2h_bytes = ex->d2h;
  }
  if (log && log_len) {
    const int64_t n = std::min<int64_t>(log_cap, (int64_t)st.log.size());
    for (int64_t i = 0; i < n; ++i) {
      const auto& a = st.log[i];
      log[i] = cs_iter_log{a.t_ms, a.pred_ms, a.ms, a.device_ms, a.c, a.s, a.phase, a.layer, a.l,
                           a.n_decode, a.n_prefill, a.n_running, a.n_queue, a.timed ? 1 : 0};
    }
    *log_len = n;
  }
  delete ex;
  return rc;
}
