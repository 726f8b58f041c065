// dpg_train.cpp — the C++ host path end to end, no Python: a DP-SGD training loop over the C ABI
// (include/dpg.h), the way a dpgrad user drives make_private -> DpOptimizer::step, here on the
// B200 engine. CIFAR-10 4-layer CNN, synthetic data, one CUDA-graph step per
// batch; prints one JSON line (samples/s, mean loss of the last step, parameter checksum).
//
//   build:  make -C paper_2109_12298_b200/csrc examples   (-> paper_2109_12298_b200/dpg_train)
//   run:    paper_2109_12298_b200/dpg_train [steps] [batch] [sigma] [C]
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "dpg.h"

#define CHECK(call)                                                                  \
  do {                                                                               \
    dpg_status st_ = (call);                                                         \
    if (st_ != DPG_OK) {                                                             \
      std::fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, dpg_last_error(ctx)); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

static dpg_layer_desc conv(int64_t ic, int64_t oc) {
  dpg_layer_desc d{};
  d.kind = DPG_LAYER_CONV2D;
  d.has_bias = 1;
  d.in_channels = ic;
  d.out_channels = oc;
  d.kernel_h = d.kernel_w = 3;
  d.stride = 2;
  d.padding = 1;
  return d;
}
static dpg_layer_desc plain(int kind) {
  dpg_layer_desc d{};
  d.kind = kind;
  return d;
}

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 200;
  const int64_t b = argc > 2 ? std::atoll(argv[2]) : 512;
  const double sigma = argc > 3 ? std::atof(argv[3]) : 1.0;
  const double clip = argc > 4 ? std::atof(argv[4]) : 1.0;
  dpg_ctx* ctx = nullptr;
  if (dpg_ctx_create(0, nullptr, &ctx) != DPG_OK) {
    std::fprintf(stderr, "dpg_ctx_create: %s\n", dpg_last_error(nullptr));
    return 1;
  }
  dpg_layer_desc fc{};
  fc.kind = DPG_LAYER_LINEAR;
  fc.has_bias = 1;
  fc.in_features = 512;
  fc.out_features = 10;
  const dpg_layer_desc layers[] = {conv(3, 32), plain(DPG_LAYER_RELU), conv(32, 64), plain(DPG_LAYER_RELU),
                                   conv(64, 64), plain(DPG_LAYER_RELU), conv(64, 128), plain(DPG_LAYER_RELU),
                                   plain(DPG_LAYER_FLATTEN), fc};
  const int nl = sizeof(layers) / sizeof(layers[0]);
  const int64_t in_shape[] = {3, 32, 32};
  dpg_model* model = nullptr;
  CHECK(dpg_model_create(ctx, layers, nl, in_shape, 3, b, &model));
  // build_model's initialisation (layers.hpp:926-973): U(+-1/sqrt(fan_in)) per parameter tensor
  const int64_t L = dpg_model_parameter_count(model);
  std::vector<float> params((size_t)L);
  std::mt19937_64 rng(1);
  for (int p = 0; p < dpg_model_num_param_tensors(model); ++p) {
    int layer = 0, slot = 0;
    int64_t numel = 0, offset = 0;
    CHECK(dpg_model_param_info(model, p, &layer, &slot, &numel, &offset));
    const dpg_layer_desc& d = layers[layer];
    const double fan_in = d.kind == DPG_LAYER_LINEAR ? (double)d.in_features
                                                     : (double)(d.in_channels * d.kernel_h * d.kernel_w);
    std::uniform_real_distribution<float> u(-1.0 / std::sqrt(fan_in), 1.0 / std::sqrt(fan_in));
    for (int64_t i = 0; i < numel; ++i) params[(size_t)(offset + i)] = u(rng);
  }
  CHECK(dpg_model_load_params(model, params.data()));
  dpg_optimizer_config cfg{sigma, clip, 0.1, (double)b, 3, 1, 0};
  dpg_optimizer* opt = nullptr;
  CHECK(dpg_optimizer_create(model, &cfg, &opt));

  // synthetic CIFAR-shaped batch, resident on the device
  std::vector<float> hx((size_t)(b * 3 * 32 * 32)), hy((size_t)b);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::uniform_int_distribution<int> cls(0, 9);
  for (auto& v : hx) v = nd(rng);
  for (auto& v : hy) v = (float)cls(rng);
  float *x = nullptr, *y = nullptr, *loss = nullptr;
  cudaMalloc(&x, sizeof(float) * hx.size());
  cudaMalloc(&y, sizeof(float) * hy.size());
  cudaMalloc(&loss, sizeof(float) * b);
  cudaMemcpy(x, hx.data(), sizeof(float) * hx.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(y, hy.data(), sizeof(float) * hy.size(), cudaMemcpyHostToDevice);

  for (int i = 0; i < 5; ++i) CHECK(dpg_train_step(opt, x, y, b, loss, 1));  // capture + warm-up
  CHECK(dpg_ctx_sync(ctx));
  cudaStream_t stream = static_cast<cudaStream_t>(dpg_ctx_stream(ctx));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, stream);
  for (int i = 0; i < steps; ++i) CHECK(dpg_train_step(opt, x, y, b, loss, 1));
  cudaEventRecord(e1, stream);
  CHECK(dpg_ctx_sync(ctx));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);

  std::vector<float> hl((size_t)b);
  cudaMemcpy(hl.data(), loss, sizeof(float) * b, cudaMemcpyDeviceToHost);
  double mean_loss = 0;
  for (float v : hl) mean_loss += v;
  mean_loss /= (double)b;
  CHECK(dpg_model_store_params(model, params.data()));
  double checksum = 0;
  for (float v : params) checksum += std::fabs((double)v);
  std::printf("{\"program\": \"dpg_train\", \"steps\": %d, \"batch\": %lld, \"samples_per_s\": %.1f, "
              "\"ms_per_step\": %.4f, \"mean_loss\": %.6f, \"param_abs_sum\": %.6f, \"finite\": %s}\n",
              steps, (long long)b, 1000.0 * steps * (double)b / ms, ms / steps, mean_loss, checksum,
              std::isfinite(checksum) && std::isfinite(mean_loss) ? "true" : "false");
  cudaFree(x);
  cudaFree(y);
  cudaFree(loss);
  dpg_optimizer_destroy(opt);
  dpg_model_destroy(model);
  dpg_ctx_destroy(ctx);
  return 0;
}
