// sched_capi.cpp -- C exports of the host cost model (include/coserve/cost_model.hpp).
#include <limits>
#include <stdexcept>
#include <string>

#include "coserve/cost_model.hpp"
#include "coserve_cuda.h"

namespace cs {
int set_error(int code, const std::string& msg);
}

namespace {
coserve::LatencyProfile to_profile(const cs_latency_profile* p) {
  coserve::LatencyProfile q;
  q.t0_ms = p->t0_ms;
  q.slope_ms_per_token = p->slope_ms_per_token;
  q.knee_tokens = p->knee_tokens > 0 ? p->knee_tokens : std::numeric_limits<double>::infinity();
  q.bwd_token_weight = p->bwd_token_weight > 0 ? p->bwd_token_weight : 1.0;
  q.attn_fwd_ms_per_token_ctx = p->attn_fwd_ms_per_token_ctx;
  q.attn_bwd_ms_per_token_ctx = p->attn_bwd_ms_per_token_ctx;
  q.bwd_layer0_weight = p->bwd_layer0_weight > 0 ? p->bwd_layer0_weight : 1.0;
  q.decode_ms_per_row = p->decode_ms_per_row > 0 ? p->decode_ms_per_row : 0.0;
  q.prefill_ms_per_token = p->prefill_ms_per_token > 0 ? p->prefill_ms_per_token : 0.0;
  q.fwd_window_ms = p->fwd_window_ms > 0 ? p->fwd_window_ms : 0.0;
  return q;
}
}  // namespace

extern "C" double cs_sched_latency(const cs_latency_profile* p, int64_t c, int64_t s) {
  if (!p || c < 0 || s < 0) return -1.0;
  return coserve::latency(to_profile(p), c, s);
}

extern "C" int64_t cs_sched_max_finetune_tokens(const cs_latency_profile* p, int64_t c,
                                                double slo_ms) {
  if (!p || c < 0 || !(slo_ms > 0)) return -1;
  return coserve::max_finetune_tokens(to_profile(p), c, slo_ms);
}
