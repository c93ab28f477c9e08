// coserve/calibrate.hpp -- online calibration of the iteration latency model f(c, s) against
// measured device time (the B200 co-serving loop's adaptive mode 2).
//
// The planner's prediction for a plan is linear in the profile coefficients
//   pred = t0 + d n_dec + f n_pre                                      (inference rows)
//        + [s_f > 0] w_f + b s_f + a_f s_f (l + s_f / 2)               (forward window)
//        + sum_windows g_y (b_b s + a_b s (l_j - s / 2))               (backward windows)
// (cost_model.hpp: inference_cost, ft_fwd_cost, ft_bwd_cost; g_y = the layer-0 weight for layer
// 0 and 1 otherwise), so one measured iteration is one linear observation of
// theta = [t0, d, f, w_f, b, a_f, b_b, a_b].  A Kalman filter with a random-walk model keeps
// theta tracking the box (clock / power state, GEMM tile quantisation the offline fit averages
// away) per coefficient; the per-phase scalar correction (adaptive mode 1) can only rescale all
// of them together, which leaves the relative miscalibration between the terms -- forward
// iterations of long vs short windows, backward windows at long vs short context -- in the
// residual, and the tail controller then has to budget for it.
#pragma once
#include <algorithm>
#include <array>
#include <cmath>

#include "coserve/cost_model.hpp"
#include "coserve/scheduler.hpp"

namespace coserve {

class CostCalibrator {
 public:
  static constexpr int K = 8;
  using Vec = std::array<double, K>;

  // usable when the profile has the per-kind row slopes and the context terms (the measured
  // B200 profile); otherwise the loop keeps the scalar correction
  static bool applicable(const LatencyProfile& p) { return p.has_ctx_terms() && p.has_row_terms(); }

  explicit CostCalibrator(const LatencyProfile& prior) : prior_(prior) {
    const double w = prior.bwd_token_weight > 0 ? prior.bwd_token_weight : 1.0;
    theta0_ = {prior.t0_ms, prior.decode_ms_per_row, prior.prefill_ms_per_token, prior.fwd_window_ms,
               prior.slope_ms_per_token, prior.attn_fwd_ms_per_token_ctx, w * prior.slope_ms_per_token,
               prior.attn_bwd_ms_per_token_ctx};
    theta_ = theta0_;
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j) P_[i][j] = i == j ? sq(kPriorRel * scale(i)) : 0.0;
  }

  // the feature vector of a plan (its prediction under theta is dot(theta, features))
  Vec features(const IterationPlan& p) const {
    Vec x{};
    x[0] = 1.0;
    const double nd = (double)p.decode.size();
    x[1] = nd;
    x[2] = (double)p.c - nd;
    if (p.ft_phase == FtPhase::Forward && p.s > 0) {
      const double s = (double)p.s;
      x[3] = 1.0;
      x[4] = s;
      x[5] = s * ((double)p.ft_l + 0.5 * s);
    } else if (p.ft_phase == FtPhase::Backward) {
      for (const BwdWindow& w : p.bwd) {
        const double g = w.layer == 0 ? prior_.bwd_layer0_weight : 1.0;
        const double s = (double)w.s;
        x[6] += g * s;
        x[7] += g * s * ((double)w.lj - 0.5 * s);
      }
    }
    return x;
  }

  double predict(const Vec& x) const {
    double y = 0;
    for (int i = 0; i < K; ++i) y += theta_[i] * x[i];
    return y;
  }

  // one measured iteration: device time y_ms of a plan with features x
  void update(const Vec& x, double y_ms) {
    if (!(y_ms > 0)) return;
    // random walk: each coefficient may drift by kDriftRel of its prior per iteration
    for (int i = 0; i < K; ++i) P_[i][i] += sq(kDriftRel * scale(i));
    Vec px{};
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j) px[i] += P_[i][j] * x[j];
    double s = sq(kNoiseRel * y_ms);
    for (int i = 0; i < K; ++i) s += x[i] * px[i];
    const double e = y_ms - predict(x);
    for (int i = 0; i < K; ++i) {
      const double k = px[i] / s;
      theta_[i] += k * e;
    }
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j) P_[i][j] -= px[i] * px[j] / s;
    // keep every coefficient within [1/2, 2] x its prior (zero priors stay zero)
    for (int i = 0; i < K; ++i) theta_[i] = std::min(2.0 * theta0_[i], std::max(0.5 * theta0_[i], theta_[i]));
  }

  // the calibrated profile the planner uses next
  LatencyProfile profile() const {
    LatencyProfile p = prior_;
    p.t0_ms = theta_[0];
    p.decode_ms_per_row = theta_[1];
    p.prefill_ms_per_token = theta_[2];
    p.fwd_window_ms = theta_[3];
    p.slope_ms_per_token = theta_[4];
    p.attn_fwd_ms_per_token_ctx = theta_[5];
    p.bwd_token_weight = theta_[4] > 0 ? theta_[6] / theta_[4] : prior_.bwd_token_weight;
    p.attn_bwd_ms_per_token_ctx = theta_[7];
    return p;
  }
  const Vec& theta() const { return theta_; }

 private:
  static double sq(double v) { return v * v; }
  double scale(int i) const { return std::fabs(theta0_[i]); }
  static constexpr double kPriorRel = 0.15;   // prior std: 15% of each profiled coefficient
  static constexpr double kDriftRel = 0.004;  // random-walk std per iteration
  static constexpr double kNoiseRel = 0.025;  // measurement noise: 2.5% of the iteration
  LatencyProfile prior_;
  Vec theta0_{}, theta_{};
  double P_[K][K] = {};
};

}  // namespace coserve
