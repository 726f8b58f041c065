// adapter_parity.cpp — the reference's own engine driving the GPU rules (TEST HARNESS).
//
// Built by oracle/Makefile against the reference sources (where /root/reference exists) and
// libdpg.so, into oracle/_ref/adapter_parity; run on the GPU box by tests/test_gpu_adapter.py.
// For the MNIST, CIFAR, embedding and a layer_norm / group_norm model it runs compute_grad_samples (grad_sample.hpp:328-343)
// twice on the same inputs — default registry vs make_gpu_registry — then one full
// make_private / DpOptimizer step each, and prints one JSON line with the max-scaled differences.
#include <cmath>
#include <cstdio>
#include <vector>

#include "dpgrad/grad_sample.hpp"
#include "dpgrad/optimizer.hpp"
#include "dpgrad_gpu_rules.hpp"

using namespace dpgrad;

static double maxscaled(const Tensor<float>& a, const Tensor<float>& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.numel(); ++i) {
    num = std::max(num, std::fabs((double)a[i] - (double)b[i]));
    den = std::max(den, std::fabs((double)b[i]));
  }
  return den > 0 ? num / den : num;
}

static ModelGraph<float> model_for(int which) {
  RngStream rng = RngStream::standard(1);
  std::vector<LayerDescriptor> d;
  if (which == 0) {
    d = {LayerDescriptor::conv2d(1, 16, 8, 8, 2, 0), LayerDescriptor::relu(), LayerDescriptor::conv2d(16, 32, 4, 4, 2, 0),
         LayerDescriptor::relu(), LayerDescriptor::flatten(), LayerDescriptor::linear(512, 32), LayerDescriptor::relu(),
         LayerDescriptor::linear(32, 10)};
  } else if (which == 1) {
    d = {LayerDescriptor::conv2d(3, 32, 3, 3, 2, 1),  LayerDescriptor::relu(), LayerDescriptor::conv2d(32, 64, 3, 3, 2, 1),
         LayerDescriptor::relu(),                     LayerDescriptor::conv2d(64, 64, 3, 3, 2, 1), LayerDescriptor::relu(),
         LayerDescriptor::conv2d(64, 128, 3, 3, 2, 1), LayerDescriptor::relu(),                     LayerDescriptor::flatten(),
         LayerDescriptor::linear(512, 10)};
  } else if (which == 2) {
    d = {LayerDescriptor::embedding(10000, 128), LayerDescriptor::flatten(), LayerDescriptor::linear(128 * 16, 2)};
  } else {
    d = {LayerDescriptor::conv2d(3, 8, 3, 3, 1, 1), LayerDescriptor::group_norm(2, 8), LayerDescriptor::relu(),
         LayerDescriptor::flatten(), LayerDescriptor::linear(8 * 6 * 6, 32), LayerDescriptor::layer_norm(Shape{32}),
         LayerDescriptor::relu(), LayerDescriptor::linear(32, 10)};
  }
  return build_model<float>(d, rng);
}

int main() {
  dpg_ctx* ctx = nullptr;
  if (dpg_ctx_create(0, nullptr, &ctx) != DPG_OK) {
    std::printf("{\"error\": \"%s\"}\n", dpg_last_error(nullptr));
    return 1;
  }
  const auto gpu_reg = dpgrad_gpu::make_gpu_registry(ctx);
  const char* names[] = {"mnist", "cifar", "embedding", "norms"};
  std::printf("{");
  double worst = 0;
  for (int which = 0; which < 4; ++which) {
    ModelGraph<float> m = model_for(which);
    const std::size_t b = 8;
    RngStream data = RngStream::standard(2);
    Tensor<float> x;
    if (which == 0) x = gaussian<float>({b, 1, 28, 28}, 1.0, data);
    else if (which == 1) x = gaussian<float>({b, 3, 32, 32}, 1.0, data);
    else if (which == 3) x = gaussian<float>({b, 3, 6, 6}, 1.0, data);
    else {
      x = Tensor<float>({b, 16});
      for (std::size_t i = 0; i < x.numel(); ++i) x[i] = (float)data.below(10000);
    }
    const std::size_t k = which == 2 ? 2 : 10;
    Tensor<float> y({b});
    for (std::size_t i = 0; i < b; ++i) y[i] = (float)data.below(k);
    EngineResult<float> ref = compute_grad_samples(m, x, y, LossKind::softmax_cross_entropy);
    EngineResult<float> gpu = compute_grad_samples(m, x, y, LossKind::softmax_cross_entropy, gpu_reg);
    double err = 0;
    for (std::size_t l = 0; l < ref.record.per_layer.size(); ++l)
      for (std::size_t p = 0; p < ref.record.per_layer[l].size(); ++p)
        err = std::max(err, maxscaled(gpu.record.per_layer[l][p], ref.record.per_layer[l][p]));
    // a whole DP step through make_private with the GPU registry vs the default one
    DpOptimizerConfig cfg;
    cfg.expected_batch_size = (double)b;
    LoaderConfig lc{0.5, 100, 7};
    ModelGraph<float> m1 = model_for(which), m2 = model_for(which);
    auto p1 = make_private(m1, cfg, lc, GradSamplerRegistry<float>::with_defaults(), 3);
    auto p2 = make_private(m2, cfg, lc, gpu_reg, 3);
    p1.optimizer.set_grad_sample(p1.module.forward_backward(x, y, LossKind::softmax_cross_entropy).record);
    p2.optimizer.set_grad_sample(p2.module.forward_backward(x, y, LossKind::softmax_cross_entropy).record);
    p1.optimizer.step();
    p2.optimizer.step();
    double perr = 0;
    for (std::size_t l = 0; l < m1.layers.size(); ++l)
      for (std::size_t p = 0; p < m1.layers[l].params.size(); ++p)
        perr = std::max(perr, maxscaled(m2.layers[l].params[p].value, m1.layers[l].params[p].value));
    std::printf("%s\"%s\": {\"record_maxscaled\": %.3e, \"params_maxscaled\": %.3e}", which ? ", " : "", names[which], err,
                perr);
    worst = std::max(worst, err);
  }
  std::printf(", \"worst_record_maxscaled\": %.3e}\n", worst);
  dpg_ctx_destroy(ctx);
  return worst <= 1e-5 ? 0 : 2;
}
