// The INTEGRATION.md example as a test: a reference user's program -- the reference headers
// unmodified (/root/reference/proj/include: TinyModel, forward_full, backward_full,
// max_rel_err) plus coserve/gpu.hpp -- runs the same model through the B200 path and checks it
// with the reference's own metric.  Compiled in the dev container (tests/test_cpp_wrapper.py,
// where the reference tree exists), executed on the GPU box (the prebuilt binary travels).
// Prints one JSON line; exit code 0 iff every check passed.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "coserve/gpu.hpp"
#include "coserve/tiny_model.hpp"

namespace {
int failures = 0;
void expect(bool ok, const char* what) {
  if (!ok) {
    std::fprintf(stderr, "FAILED: %s\n", what);
    ++failures;
  }
}
double scaled(const coserve::Matrix& a, const coserve::Matrix& b) {  // max|a-b| / max|b|
  double m = 0, s = 1e-30;
  for (std::size_t i = 0; i < a.data().size(); ++i) {
    m = std::max(m, std::fabs(a.data()[i] - b.data()[i]));
    s = std::max(s, std::fabs(b.data()[i]));
  }
  return m / s;
}
}  // namespace

int main() {
  using namespace coserve;
  // --- BEGIN INTEGRATION EXAMPLE ---
  TinyModelConfig cfg;          // SURVEY Appendix A cfg B = BASELINE config 1
  cfg.depth = 2;
  cfg.hidden = 256;
  cfg.heads = 4;
  cfg.vocab = 64;
  cfg.lora_rank = 8;
  cfg.seed = 1;
  TinyModel m = TinyModel::init(cfg);                       // reference init, unchanged
  Rng rng(42);
  std::vector<int> tokens;
  for (int i = 0; i < 64; ++i) tokens.push_back((int)rng.uniform_int(0, cfg.vocab - 1));

  ForwardTrace tr = forward_full(m, tokens);                 // reference, CPU f64
  OracleResult ref = backward_full(m, tr);

  gpu::Engine eng = gpu::Engine::from_tiny_model(m, /*max_ft_len=*/64);   // B200
  gpu::GpuResult res = gpu::forward_backward_full(eng, tokens, /*fwd_window=*/20,
                                                  /*bwd_window=*/24);
  LoraGrads g;
  for (int l = 0; l < cfg.depth; ++l) {
    g.a.push_back(res.grad_a[l].to<Matrix>());
    g.b.push_back(res.grad_b[l].to<Matrix>());
  }
  const double grad_err = max_grad_rel_err(g, ref.grads);   // the reference's own metric
  // --- END INTEGRATION EXAMPLE ---
  expect(rel_err(res.loss, tr.loss) < 1e-2, "loss rel_err < 1e-2");
  expect(grad_err < 1e-2, "max_grad_rel_err < 1e-2");
  // scale-normalised (an all-zero gradient scores 1): top layer at the bf16 floor (2%),
  // layer 0 behind the ReLU-mask-chaotic dX (8%; tests/test_coserve_gpu.py)
  const double sa1 = scaled(g.a[1], ref.grads.a[1]), sb1 = scaled(g.b[1], ref.grads.b[1]);
  const double sa0 = scaled(g.a[0], ref.grads.a[0]), sb0 = scaled(g.b[0], ref.grads.b[0]);
  expect(sa1 < 0.02 && sb1 < 0.02, "top-layer LoRA grads within 2% scale-normalised");
  expect(sa0 < 0.08 && sb0 < 0.08, "layer-0 LoRA grads within 8% scale-normalised");
  const double sdk = scaled(res.layers[1].dk.to<Matrix>(), ref.layers[1].dk);
  const double sdv = scaled(res.layers[1].dv.to<Matrix>(), ref.layers[1].dv);
  const double sdx = scaled(res.layers[1].dx.to<Matrix>(), ref.layers[1].dx);
  expect(sdk < 0.08 && sdv < 0.08 && sdx < 0.08, "layer-1 dK/dV/dX within 8% scale-normalised");
  expect(res.layers[0].dk.empty(), "layer 0 forms no dK (graph pruning)");

  // error conventions
  bool threw = false;
  try {
    TinyModelConfig bad = cfg;
    bad.hidden = 16;  // head_dim 4: not a supported head dimension
    gpu::Engine::from_tiny_model(TinyModel::init(bad), 64);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  expect(threw, "unsupported config -> std::invalid_argument");
  gpu::QkvCache c = eng.make_cache(64);
  eng.reset_finetuning();
  threw = false;
  try {
    gpu::forward_window(eng, tokens, /*l_i=*/2, /*s=*/2, c);   // cache is empty: SPEC.md:287
  } catch (const gpu::CacheDesync&) {
    threw = true;
  }
  expect(threw, "forward_window at l_i != cache length -> CacheDesync");
  threw = false;
  try {
    gpu::forward_window(eng, tokens, 0, 64, c);
    gpu::backward_window(eng, /*n=*/0, 64, 8, c);              // top layer first: SPEC.md:296
  } catch (const gpu::OrderingViolation&) {
    threw = true;
  }
  expect(threw, "backward_window out of order -> OrderingViolation");

  std::printf("{\"loss_gpu\": %.9g, \"loss_ref\": %.9g, \"max_grad_rel_err\": %.6g, "
              "\"scaled\": {\"dA1\": %.5g, \"dB1\": %.5g, \"dA0\": %.5g, \"dB0\": %.5g, "
              "\"dK1\": %.5g, \"dV1\": %.5g, \"dX1\": %.5g}, \"failures\": %d}\n",
              res.loss, tr.loss, grad_err, sa1, sb1, sa0, sb0, sdk, sdv, sdx, failures);
  return failures == 0 ? 0 : 1;
}
