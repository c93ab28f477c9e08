// coserve/workload.hpp -- synthetic arrivals: inhomogeneous Poisson with
// sinusoidally modulated rate lambda(t) = rate * (1 + a * sin(2 pi t / period)), lognormal
// prompt / generation lengths clipped to [16, 4096] / [8, 1024], deterministic
// given the seed.  Rng follows the reference's hand-rolled distributions over mt19937_64
// (rng.hpp:15-64) so traces are reproducible bit-for-bit across implementations.
#pragma once
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <vector>

namespace coserve {

class TraceRng {
 public:
  explicit TraceRng(uint64_t seed) : eng_(seed) {}
  double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  int64_t uniform_int(int64_t lo, int64_t hi) {
    return lo + static_cast<int64_t>(eng_() % static_cast<uint64_t>(hi - lo + 1));
  }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare_ = r * std::sin(th);
    have_spare_ = true;
    return r * std::cos(th);
  }
  double lognormal(double mu, double sigma) { return std::exp(mu + sigma * normal()); }
  double exponential(double rate) {
    double u = uniform();
    while (u <= 0.0) u = uniform();
    return -std::log(u) / rate;
  }

 private:
  std::mt19937_64 eng_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

struct Arrival {
  double time_ms = 0.0;
  int tenant = 0;
  int prompt_len = 1;
  int gen_len = 1;
};

struct WorkloadConfig {
  double rate_rps = 20.0;
  double duration_s = 60.0;
  double burst_amplitude = 0.0;  // a in [0, 1]
  double burst_period_s = 60.0;
  double prompt_mu = 5.5, prompt_sigma = 0.8;
  int prompt_min = 16, prompt_max = 4096;
  double gen_mu = 4.5, gen_sigma = 0.7;
  int gen_min = 8, gen_max = 1024;
  // tenants (VTC fairness runs): arrival i goes to tenant 0 with probability tenant0_share,
  // else uniformly to 1..n_tenants-1; drawn from a separate stream, so times and lengths are
  // the single-tenant trace's
  int n_tenants = 1;
  double tenant0_share = 0.5;
};

inline int clip_len(double v, int lo, int hi) {
  const long r = std::lround(v);
  return (int)std::max<long>(lo, std::min<long>(hi, r));
}

// SPEC.md:635-643 (thinning; draw order per arrival: gap, accept, prompt, gen)
inline std::vector<Arrival> generate_trace(const WorkloadConfig& c, uint64_t seed) {
  if (c.burst_amplitude < 0 || c.burst_amplitude > 1)
    throw std::invalid_argument("generate_trace: amplitude must be in [0, 1]");
  std::vector<Arrival> out;
  if (c.rate_rps <= 0 || c.duration_s <= 0) return out;
  TraceRng rng(seed);
  const double lam_max = c.rate_rps * (1.0 + c.burst_amplitude);
  double t = 0.0;  // seconds
  while (true) {
    t += rng.exponential(lam_max);
    if (t >= c.duration_s) break;
    const double lam = c.rate_rps * (1.0 + c.burst_amplitude *
                                               std::sin(2.0 * M_PI * t / c.burst_period_s));
    const double u = rng.uniform();
    if (u * lam_max > lam) continue;
    Arrival a;
    a.time_ms = t * 1000.0;
    a.prompt_len = clip_len(rng.lognormal(c.prompt_mu, c.prompt_sigma), c.prompt_min, c.prompt_max);
    a.gen_len = clip_len(rng.lognormal(c.gen_mu, c.gen_sigma), c.gen_min, c.gen_max);
    out.push_back(a);
  }
  if (c.n_tenants > 1) {
    TraceRng trng(seed ^ 0x7E7A7E7Aull);
    for (auto& a : out) {
      const double u = trng.uniform();
      a.tenant = u < c.tenant0_share ? 0 : 1 + (int)trng.uniform_int(0, c.n_tenants - 2);
    }
  }
  return out;
}

// SPEC.md:644-652
inline std::vector<Arrival> rescale(std::vector<Arrival> tr, double factor) {
  if (!(factor > 0)) throw std::invalid_argument("rescale: factor must be > 0");
  for (auto& a : tr) a.time_ms /= factor;
  return tr;
}

}  // namespace coserve
