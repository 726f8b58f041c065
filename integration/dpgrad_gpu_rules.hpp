// dpgrad_gpu_rules.hpp — drop-in GPU rules for the reference's plugin API.
//
// The reference drives per-sample gradients through GradSamplerRegistry (grad_sample.hpp:156-238):
// a rule key -> std::function<vector<Tensor<T>>(const Layer<T>&, const LayerCache<T>&,
// const Tensor<T>& highway)>, looked up by the backward walk (grad_sample.hpp:291-292). This
// header builds a registry whose "linear", "conv2d", "embedding", "layer_norm" and "group_norm"
// rules run on the B200 through
// the C ABI (include/dpg.h), registered with override_existing = true (grad_sample.hpp:159-167),
// so compute_grad_samples / GradSampleModule / make_private work unchanged:
//
//     dpg_ctx* ctx; dpg_ctx_create(0, nullptr, &ctx);
//     auto reg = dpgrad_gpu::make_gpu_registry(ctx);
//     auto priv = dpgrad::make_private(model, cfg, loader, reg);      // unchanged caller
//
// Each rule call copies the layer's cached input and highway to the device, runs the rule, and
// copies the per-sample gradients back (the reference's record lives in host Tensors). This is the
// parity path; the throughput path is the device-resident engine ABI (dpg_forward_backward /
// dpg_step), which keeps everything in HBM.
//
// Status codes are rethrown as the matching dpgrad exception (errors.hpp:12-72).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "dpg.h"
#include "dpgrad/errors.hpp"
#include "dpgrad/grad_sample.hpp"

namespace dpgrad_gpu {

inline void check(dpg_status st, dpg_ctx* ctx) {
  if (st == DPG_OK) return;
  const std::string msg = dpg_last_error(ctx);
  switch (st) {
    case DPG_ERR_DIMENSION: throw dpgrad::DimensionError(msg);
    case DPG_ERR_PARAMETER: throw dpgrad::ParameterError(msg);
    case DPG_ERR_LIFECYCLE: throw dpgrad::LifecycleError(msg);
    case DPG_ERR_REGISTRY: throw dpgrad::RegistryError(msg);
    case DPG_ERR_NUMERIC: throw dpgrad::NumericError(msg);
    default: throw dpgrad::Error("libdpg: " + msg);
  }
}

// Device scratch owned by one rule invocation.
struct DevBuf {
  float* p = nullptr;
  size_t n = 0;
  explicit DevBuf(size_t count) : n(count) {
    if (count && cudaMalloc(&p, count * sizeof(float)) != cudaSuccess)
      throw dpgrad::Error("cudaMalloc failed");
  }
  DevBuf(const float* host, size_t count) : DevBuf(count) {
    if (count) cudaMemcpy(p, host, count * sizeof(float), cudaMemcpyHostToDevice);
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void to_host(float* host) const {
    if (n) cudaMemcpy(host, p, n * sizeof(float), cudaMemcpyDeviceToHost);
  }
};

inline dpgrad::GradSamplerRegistry<float> make_gpu_registry(dpg_ctx* ctx) {
  using namespace dpgrad;
  auto reg = GradSamplerRegistry<float>::with_defaults();
  // registry "linear" (grad_sample.hpp:188-201)
  reg.register_rule(
      "linear",
      [ctx](const Layer<float>& layer, const LayerCache<float>& cache, const Tensor<float>& hw) {
        const std::size_t d = layer.desc.in_features, r = layer.desc.out_features;
        const std::size_t b = cache.input.extent(0), mid = cache.input.numel() / (b * d);
        DevBuf a(cache.input.data(), cache.input.numel()), h(hw.data(), hw.numel());
        DevBuf gw(b * r * d), gb(layer.desc.has_bias ? b * r : 0);
        check(dpg_grad_sample_linear(ctx, a.p, h.p, (int64_t)b, (int64_t)mid, (int64_t)d, (int64_t)r,
                                     gw.p, layer.desc.has_bias ? gb.p : nullptr, nullptr, nullptr),
              ctx);
        check(dpg_ctx_sync(ctx), ctx);
        std::vector<Tensor<float>> out;
        out.emplace_back(Shape{b, r, d});
        gw.to_host(out.back().data());
        if (layer.desc.has_bias) {
          out.emplace_back(Shape{b, r});
          gb.to_host(out.back().data());
        }
        return out;
      },
      /*override_existing=*/true);
  // registry "conv2d" (grad_sample.hpp:208-215)
  reg.register_rule(
      "conv2d",
      [ctx](const Layer<float>& layer, const LayerCache<float>& cache, const Tensor<float>& hw) {
        const Conv2dSpec& c = layer.desc.conv;
        const std::size_t b = cache.input.extent(0), h = cache.input.extent(2), w = cache.input.extent(3);
        const dpg_conv2d_spec spec{(int64_t)c.in_channels, (int64_t)c.out_channels, (int64_t)c.kernel_h,
                                   (int64_t)c.kernel_w,    (int64_t)c.stride,       (int64_t)c.padding};
        const std::size_t k = c.in_channels * c.kernel_h * c.kernel_w;
        DevBuf x(cache.input.data(), cache.input.numel()), hd(hw.data(), hw.numel());
        DevBuf gw(b * c.out_channels * k), gb(layer.desc.has_bias ? b * c.out_channels : 0);
        check(dpg_grad_sample_conv2d(ctx, x.p, hd.p, (int64_t)b, (int64_t)h, (int64_t)w, &spec, gw.p,
                                     layer.desc.has_bias ? gb.p : nullptr, nullptr, nullptr),
              ctx);
        check(dpg_ctx_sync(ctx), ctx);
        std::vector<Tensor<float>> out;
        out.emplace_back(Shape{b, c.out_channels, c.in_channels, c.kernel_h, c.kernel_w});
        gw.to_host(out.back().data());
        if (layer.desc.has_bias) {
          out.emplace_back(Shape{b, c.out_channels});
          gb.to_host(out.back().data());
        }
        return out;
      },
      true);
  // registry "embedding" (grad_sample.hpp:202-207)
  reg.register_rule(
      "embedding",
      [ctx](const Layer<float>& layer, const LayerCache<float>& cache, const Tensor<float>& hw) {
        const std::size_t b = cache.input.extent(0), t = cache.input.extent(1);
        const std::size_t v = layer.desc.vocab_size, d = layer.desc.embedding_dim;
        DevBuf idx(cache.input.data(), cache.input.numel()), hd(hw.data(), hw.numel());
        DevBuf g(b * v * d);
        check(dpg_grad_sample_embedding(ctx, idx.p, hd.p, (int64_t)b, (int64_t)t, (int64_t)v, (int64_t)d, g.p,
                                        nullptr),
              ctx);
        check(dpg_ctx_sync(ctx), ctx);  // surfaces out-of-range indices as ParameterError
        std::vector<Tensor<float>> out;
        out.emplace_back(Shape{b, v, d});
        g.to_host(out.back().data());
        return out;
      },
      true);
  // registry "layer_norm" / "group_norm" (grad_sample.hpp:216-225): the rules read the forward
  // cache's normalized input (layers.hpp:249-262)
  auto norm_rule = [ctx](bool group) {
    return [ctx, group](const Layer<float>& layer, const LayerCache<float>& cache, const Tensor<float>& hw) {
      const std::size_t b = cache.input.extent(0);
      const std::size_t c = group ? layer.desc.channels : shape_numel(layer.desc.normalized_shape);
      const std::size_t q = cache.input.numel() / (b * c);
      DevBuf xh(cache.normalized.data(), cache.normalized.numel()), hd(hw.data(), hw.numel());
      DevBuf gg(b * c), gb(b * c);
      check(group ? dpg_grad_sample_group_norm(ctx, xh.p, hd.p, (int64_t)b, (int64_t)c, (int64_t)q, gg.p, gb.p,
                                               nullptr, nullptr)
                  : dpg_grad_sample_layer_norm(ctx, xh.p, hd.p, (int64_t)b, (int64_t)q, (int64_t)c, gg.p, gb.p,
                                               nullptr, nullptr),
            ctx);
      check(dpg_ctx_sync(ctx), ctx);
      Shape gshape = group ? Shape{layer.desc.channels} : layer.desc.normalized_shape;
      gshape.insert(gshape.begin(), b);
      std::vector<Tensor<float>> out;
      out.emplace_back(gshape);
      gg.to_host(out.back().data());
      out.emplace_back(gshape);
      gb.to_host(out.back().data());
      return out;
    };
  };
  reg.register_rule("layer_norm", norm_rule(false), true);
  reg.register_rule("group_norm", norm_rule(true), true);
  return reg;
}

}  // namespace dpgrad_gpu
