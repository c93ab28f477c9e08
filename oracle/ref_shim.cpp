// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim around the UNMODIFIED reference headers
// (/root/reference/proj/include/coserve/{matrix,rng,tiny_model}.hpp), compiled
// by oracle/Makefile straight from where they lie into oracle/_ref/libcoserve_ref.so.
// Nothing from the reference is copied into this repository: this file only
// #includes the headers and marshals flat double buffers across the boundary.
//
// Exposes:
//   - TinyModel::init (tiny_model.hpp:44-67) and weight export,
//   - forward_full (tiny_model.hpp:181-221) + backward_full (:259-327),
//   - Rng streams (rng.hpp:15-64),
// so tests can (1) pin oracle/coserve_oracle.py against the reference itself and
// (2) time the reference CPU path for bench.py's cpu_baseline / --impl reference.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "coserve/tiny_model.hpp"

using coserve::Matrix;
using coserve::TinyModel;
using coserve::TinyModelConfig;

namespace {
thread_local std::string g_err;

void put(const Matrix& m, double* out) {
  if (out) std::memcpy(out, m.data().data(), m.data().size() * sizeof(double));
}
void get(Matrix& m, const double* in) {
  if (in) std::memcpy(m.data().data(), in, m.data().size() * sizeof(double));
}
Matrix* select(TinyModel* m, const char* name, int layer) {
  std::string n(name);
  if (n == "embed") return &m->embed;
  if (n == "unembed") return &m->unembed;
  if (layer < 0 || layer >= (int)m->layers.size()) return nullptr;
  auto& w = m->layers[layer];
  if (n == "wq") return &w.wq;
  if (n == "wk") return &w.wk;
  if (n == "wv") return &w.wv;
  if (n == "wo") return &w.wo;
  if (n == "w_up") return &w.w_up;
  if (n == "w_down") return &w.w_down;
  if (n == "lora_a") return &w.lora_a;
  if (n == "lora_b") return &w.lora_b;
  return nullptr;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Returns nullptr and sets ref_last_error() on std::invalid_argument (tiny_model.hpp:45-47).
void* ref_model_init(int depth, long hidden, int heads, long ffn_mult, long vocab, int rank,
                     uint64_t seed) {
  TinyModelConfig cfg;
  cfg.depth = depth;
  cfg.hidden = hidden;
  cfg.heads = heads;
  cfg.ffn_mult = ffn_mult;
  cfg.vocab = vocab;
  cfg.lora_rank = rank;
  cfg.seed = seed;
  try {
    return new TinyModel(TinyModel::init(cfg));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_model_free(void* h) { delete static_cast<TinyModel*>(h); }

// Copy a weight matrix out of (or into) the reference model. Returns element count or -1.
long ref_model_get(void* h, const char* name, int layer, double* out) {
  Matrix* m = select(static_cast<TinyModel*>(h), name, layer);
  if (!m) return -1;
  put(*m, out);
  return (long)m->data().size();
}
long ref_model_set(void* h, const char* name, int layer, const double* in) {
  Matrix* m = select(static_cast<TinyModel*>(h), name, layer);
  if (!m) return -1;
  get(*m, in);
  return (long)m->data().size();
}

// forward_full + backward_full. Any output pointer may be null.
//   logits [L,V]; final_hidden [L,h]; grad_a [depth][f,r]; grad_b [depth][r,h];
//   dk,dv,dx [depth][L,h]. Returns 0 ok, -1 on exception (message in ref_last_error).
int ref_forward_backward(void* h, const int* tokens, long L, double* loss, double* logits,
                         double* final_hidden, double* grad_a, double* grad_b, double* dk,
                         double* dv, double* dx) {
  try {
    const TinyModel& m = *static_cast<TinyModel*>(h);
    std::vector<int> toks(tokens, tokens + L);
    coserve::ForwardTrace tr = coserve::forward_full(m, toks);
    if (loss) *loss = tr.loss;
    put(tr.logits, logits);
    put(tr.final_hidden, final_hidden);
    if (!(grad_a || grad_b || dk || dv || dx)) return 0;
    coserve::OracleResult res = coserve::backward_full(m, tr);
    const long f = m.cfg.ffn(), r = m.cfg.lora_rank, hd = m.cfg.hidden;
    for (int l = 0; l < m.cfg.depth; ++l) {
      if (grad_a) put(res.grads.a[l], grad_a + (size_t)l * f * r);
      if (grad_b) put(res.grads.b[l], grad_b + (size_t)l * r * hd);
      if (dk) put(res.layers[l].dk, dk + (size_t)l * L * hd);
      if (dv) put(res.layers[l].dv, dv + (size_t)l * L * hd);
      if (dx) put(res.layers[l].dx, dx + (size_t)l * L * hd);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Wall time (seconds) of `iters` forward_full+backward_full calls (CPU baseline).
double ref_time_forward_backward(void* h, const int* tokens, long L, int iters) {
  const TinyModel& m = *static_cast<TinyModel*>(h);
  std::vector<int> toks(tokens, tokens + L);
  auto t0 = std::chrono::steady_clock::now();
  double sink = 0.0;
  for (int i = 0; i < iters; ++i) {
    coserve::ForwardTrace tr = coserve::forward_full(m, toks);
    coserve::OracleResult res = coserve::backward_full(m, tr);
    sink += res.loss;
  }
  auto t1 = std::chrono::steady_clock::now();
  if (sink == 12345.6789) g_err = "";
  return std::chrono::duration<double>(t1 - t0).count();
}

// Rng streams (rng.hpp:22-58).
void ref_rng_uniform_int(uint64_t seed, long n, long lo, long hi, int64_t* out) {
  coserve::Rng rng(seed);
  for (long i = 0; i < n; ++i) out[i] = rng.uniform_int(lo, hi);
}
void ref_rng_normal(uint64_t seed, long n, double* out) {
  coserve::Rng rng(seed);
  for (long i = 0; i < n; ++i) out[i] = rng.normal();
}
void ref_rng_mixed(uint64_t seed, long n, double* out) {
  // interleaves every distribution so draw-order bugs in the restatement show up
  coserve::Rng rng(seed);
  for (long i = 0; i < n; ++i) {
    switch (i % 5) {
      case 0: out[i] = rng.uniform(); break;
      case 1: out[i] = rng.normal(); break;
      case 2: out[i] = rng.lognormal(5.5, 0.8); break;
      case 3: out[i] = rng.exponential(4.0); break;
      default: out[i] = (double)rng.uniform_int(0, 63); break;
    }
  }
}

}  // extern "C"
