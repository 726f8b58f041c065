// ref_shim.cpp — C entry points over the REAL reference (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile against the reference's own headers and sources where they lie
// (/root/reference/proj/core, read-only; nothing is copied) into oracle/_ref/libdpgref.so.
// It exposes the same signatures as the C restatement (oracle/dpg_oracle.h, prefix dpgref_)
// so tests can pin the restatement bit-for-bit against the reference, and so bench.py can time
// the reference's own CPU path (`--impl reference`, cpu_baseline kind "reference").
//
// Only the reference's public API is used: build_model, compute_grad_samples,
// per_sample_rule_*, clip_and_sum, add_noise, DpOptimizer, RngStream, microbatch_oracle.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "dpgrad/grad_sample.hpp"
#include "dpgrad/layers.hpp"
#include "dpgrad/optimizer.hpp"
#include "dpgrad/rng.hpp"
#include "dpgrad/tensor.hpp"

namespace {

using namespace dpgrad;

thread_local std::string g_err;

struct CLayer {  // identical layout to dpgo_layer / dpg_layer_desc
  int32_t kind;
  int32_t has_bias;
  int64_t in_features, out_features;
  int64_t vocab_size, embedding_dim;
  int64_t in_channels, out_channels, kernel_h, kernel_w, stride, padding;
  int64_t norm_size, groups;
  double eps;
};

int code_of(const std::exception& e) {
  if (dynamic_cast<const DimensionError*>(&e)) return 1;
  if (dynamic_cast<const ParameterError*>(&e)) return 2;
  if (dynamic_cast<const LifecycleError*>(&e)) return 3;
  if (dynamic_cast<const RegistryError*>(&e)) return 4;
  if (dynamic_cast<const NumericError*>(&e)) return 5;
  return 9;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

std::vector<LayerDescriptor> descs_of(const CLayer* layers, int n) {
  std::vector<LayerDescriptor> out;
  for (int i = 0; i < n; ++i) {
    const CLayer& c = layers[i];
    switch (c.kind) {
      case 0: out.push_back(LayerDescriptor::linear(c.in_features, c.out_features, c.has_bias)); break;
      case 1: out.push_back(LayerDescriptor::embedding(c.vocab_size, c.embedding_dim)); break;
      case 2:
        out.push_back(LayerDescriptor::conv2d(c.in_channels, c.out_channels, c.kernel_h, c.kernel_w,
                                              c.stride, c.padding, c.has_bias));
        break;
      case 3: out.push_back(LayerDescriptor::layer_norm(Shape{(std::size_t)c.norm_size}, c.eps)); break;
      case 4: out.push_back(LayerDescriptor::group_norm(c.groups, c.norm_size, c.eps)); break;
      case 5: out.push_back(LayerDescriptor::relu()); break;
      case 6: out.push_back(LayerDescriptor::flatten()); break;
      default: throw ParameterError("ref_shim: unsupported layer kind");
    }
  }
  return out;
}

template <typename T>
ModelGraph<T> model_of(const CLayer* layers, int n, const T* params) {
  RngStream rng = RngStream::standard(0);
  ModelGraph<T> m = build_model<T>(descs_of(layers, n), rng);
  std::size_t off = 0;
  for (auto& layer : m.layers)
    for (auto& p : layer.params) {
      std::memcpy(p.value.data(), params + off, sizeof(T) * p.value.numel());
      off += p.value.numel();
    }
  return m;
}

template <typename T>
void copy_out(const ModelGraph<T>& m, T* params) {
  std::size_t off = 0;
  for (const auto& layer : m.layers)
    for (const auto& p : layer.params) {
      std::memcpy(params + off, p.value.data(), sizeof(T) * p.value.numel());
      off += p.value.numel();
    }
}

template <typename T>
Tensor<T> tensor_of(Shape shape, const T* data) {
  Tensor<T> t(std::move(shape));
  std::memcpy(t.data(), data, sizeof(T) * t.numel());
  return t;
}

template <typename T>
void flatten_into(const std::vector<std::vector<Tensor<T>>>& v, T* dst) {
  std::size_t off = 0;
  for (const auto& l : v)
    for (const auto& t : l) {
      std::memcpy(dst + off, t.data(), sizeof(T) * t.numel());
      off += t.numel();
    }
}

// One logical step through the reference's own optimizer (optimizer.hpp:138-278), with the
// physical batch split into `shards` virtual steps (the multi-GPU oracle).
template <typename T>
void dpsgd_step(const CLayer* layers, int nlayers, const int64_t* in_shape, int in_rank, int64_t b,
                const int64_t* shard_sizes, int nshards, T* params, const T* x, const T* targets,
                double sigma, double c, double lr, double e, uint64_t seed, const T* injected,
                T* record, T* summed, T* grad, double* norms, double* scales, int64_t* num_clipped,
                T* loss, T* logits) {
  ModelGraph<T> model = model_of<T>(layers, nlayers, params);
  DpOptimizerConfig cfg;
  cfg.noise_multiplier = injected ? 0.0 : sigma;
  cfg.max_grad_norm = c;
  cfg.learning_rate = lr;
  cfg.expected_batch_size = e;
  DpOptimizer<T> opt(model, cfg, RngStream::standard(seed));
  std::vector<int64_t> shards;
  if (shard_sizes) shards.assign(shard_sizes, shard_sizes + nshards);
  else shards.push_back(b);
  std::size_t per = 1;
  for (int i = 0; i < in_rank; ++i) per *= static_cast<std::size_t>(in_shape[i]);
  const std::size_t L = model.parameter_count();
  int64_t row0 = 0, clipped = 0;
  // index of the last non-empty shard closes the logical batch with step()
  int last = -1;
  for (int s = 0; s < static_cast<int>(shards.size()); ++s)
    if (shards[s] > 0) last = s;
  for (int s = 0; s < static_cast<int>(shards.size()); ++s) {
    const int64_t bs = shards[s];
    if (bs == 0) continue;
    Shape xs{static_cast<std::size_t>(bs)};
    for (int i = 0; i < in_rank; ++i) xs.push_back(static_cast<std::size_t>(in_shape[i]));
    Tensor<T> xt = tensor_of<T>(xs, x + row0 * per);
    Tensor<T> yt = tensor_of<T>({static_cast<std::size_t>(bs)}, targets + row0);
    EngineResult<T> res = compute_grad_samples(model, xt, yt, LossKind::softmax_cross_entropy);
    if (loss) std::memcpy(loss + row0, res.per_sample_loss.data(), sizeof(T) * bs);
    if (logits) {
      const std::size_t k = res.output.numel() / bs;
      std::memcpy(logits + row0 * k, res.output.data(), sizeof(T) * res.output.numel());
    }
    if (record) {
      std::size_t off = 0;
      for (const auto& l : res.record.per_layer)
        for (const auto& t : l) {
          const std::size_t pn = t.numel() / bs;
          std::memcpy(record + b * off + row0 * pn, t.data(), sizeof(T) * t.numel());
          off += pn;
        }
    }
    opt.set_grad_sample(std::move(res.record));
    ClipSummary cs;
    if (s == last) {
      opt.step();
      cs = opt.last_clip_summary();
    } else {
      cs = opt.virtual_step();
    }
    if (norms) std::memcpy(norms + row0, cs.per_sample_norms.data(), sizeof(double) * bs);
    if (scales) std::memcpy(scales + row0, cs.scale_factors.data(), sizeof(double) * bs);
    clipped += static_cast<int64_t>(cs.num_clipped);
    row0 += bs;
  }
  if (last < 0) opt.step_empty_batch();
  const GradientState<T>& st = opt.state();
  if (summed && st.summed_grad) flatten_into(*st.summed_grad, summed);
  if (injected) {
    // add the caller's noise tensor instead of drawing: noised = summed + noise, then the same
    // average-and-update as finish_step (optimizer.hpp:259-267) on the pre-step parameters.
    std::vector<T> flat(L);
    flatten_into(*st.summed_grad, flat.data());
    const T denom = static_cast<T>(e), lrt = static_cast<T>(lr);
    for (std::size_t i = 0; i < L; ++i) {
      const T noised = flat[i] + injected[i];
      const T g = noised * (T(1) / denom);
      params[i] = params[i] - g * lrt;
      if (grad) grad[i] = g;
    }
  } else {
    if (grad && st.grad) flatten_into(*st.grad, grad);
    copy_out(model, params);
  }
  if (num_clipped) *num_clipped = clipped;
}

// Sample-sharded host thread pool over the reference's public functions (BASELINE.md §3.1
// step 5): each thread runs compute_grad_samples + clip_and_sum on a contiguous shard, the
// main thread sums the shard outputs in shard order (virtual-step semantics), then add_noise
// and the update exactly as finish_step does.
template <typename T>
void dpsgd_step_threads(const CLayer* layers, int nlayers, const int64_t* in_shape, int in_rank,
                        int64_t b, int nthreads, T* params, const T* x, const T* targets,
                        double sigma, double c, double lr, double e, uint64_t seed) {
  const ModelGraph<T> model = model_of<T>(layers, nlayers, params);
  std::size_t per = 1;
  for (int i = 0; i < in_rank; ++i) per *= static_cast<std::size_t>(in_shape[i]);
  nthreads = std::max(1, std::min<int>(nthreads, static_cast<int>(b)));
  std::vector<SummedGrads<T>> parts(nthreads);
  std::vector<std::string> errs(nthreads);
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) {
    pool.emplace_back([&, t] {
      const int64_t lo = b * t / nthreads, hi = b * (t + 1) / nthreads;
      if (hi <= lo) return;
      try {
        Shape xs{static_cast<std::size_t>(hi - lo)};
        for (int i = 0; i < in_rank; ++i) xs.push_back(static_cast<std::size_t>(in_shape[i]));
        Tensor<T> xt = tensor_of<T>(xs, x + lo * per);
        Tensor<T> yt = tensor_of<T>({static_cast<std::size_t>(hi - lo)}, targets + lo);
        EngineResult<T> res = compute_grad_samples(model, xt, yt, LossKind::softmax_cross_entropy);
        parts[t] = clip_and_sum(res.record, c).first;
      } catch (const std::exception& ex) {
        errs[t] = ex.what();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (const auto& m : errs)
    if (!m.empty()) throw NumericError(m);
  SummedGrads<T> acc;
  for (auto& p : parts) {
    if (p.empty()) continue;
    if (acc.empty()) {
      acc = std::move(p);
      continue;
    }
    for (std::size_t l = 0; l < acc.size(); ++l)
      for (std::size_t k = 0; k < acc[l].size(); ++k) acc[l][k] = add(acc[l][k], p[l][k]);
  }
  RngStream rng = RngStream::standard(seed);
  SummedGrads<T> noised = add_noise(acc, sigma, c, rng);
  const T denom = static_cast<T>(e), lrt = static_cast<T>(lr);
  std::size_t off = 0;
  for (const auto& l : noised)
    for (const auto& t : l) {
      for (std::size_t i = 0; i < t.numel(); ++i) {
        const T g = t[i] * (T(1) / denom);
        params[off + i] = params[off + i] - g * lrt;
      }
      off += t.numel();
    }
}

}  // namespace

extern "C" {

const char* dpgref_last_error() { return g_err.c_str(); }

// the reference's NoiseSchedule (optimizer.hpp:280-358): build it with the factory of `kind`
// (0 constant, 1 exponential, 2 step, 3 custom) and evaluate schedule_noise at each epoch
int dpgref_schedule_sigmas(int kind, double sigma0, double gamma, double factor, uint64_t period,
                           const double* table, int64_t table_len, const uint64_t* epochs, int64_t n,
                           double* out) {
  return guarded([&] {
    NoiseSchedule s;
    switch (kind) {
      case 0: s = NoiseSchedule::constant(sigma0); break;
      case 1: s = NoiseSchedule::exponential(sigma0, gamma); break;
      case 2: s = NoiseSchedule::step(sigma0, factor, (std::size_t)period); break;
      default: s = NoiseSchedule::custom(std::vector<double>(table, table + table_len)); break;
    }
    for (int64_t i = 0; i < n; ++i) out[i] = schedule_noise(s, (std::size_t)epochs[i]);
  });
}

int dpgref_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  return guarded([&] {
    RngStream r = RngStream::standard(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
  });
}

int dpgref_rng_normal(uint64_t seed, int64_t n, double* out) {
  return guarded([&] {
    RngStream r = RngStream::standard(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
  });
}

int dpgref_rng_below(uint64_t seed, int64_t n, uint64_t bound, uint64_t* out) {
  return guarded([&] {
    RngStream r = RngStream::standard(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.below(bound);
  });
}

#define DPGREF_INSTANTIATE(T, SFX)                                                                 \
  int dpgref_gaussian##SFX(uint64_t seed, int64_t n, double std_dev, T* out) {                    \
    return guarded([&] {                                                                           \
      RngStream r = RngStream::standard(seed);                                                     \
      Tensor<T> t = gaussian<T>({static_cast<std::size_t>(n)}, std_dev, r);                        \
      std::memcpy(out, t.data(), sizeof(T) * n);                                                   \
    });                                                                                            \
  }                                                                                                \
  int dpgref_build_params##SFX(const CLayer* layers, int nlayers, uint64_t seed, T* params) {     \
    return guarded([&] {                                                                           \
      RngStream r = RngStream::standard(seed);                                                     \
      ModelGraph<T> m = build_model<T>(descs_of(layers, nlayers), r);                              \
      copy_out(m, params);                                                                         \
    });                                                                                            \
  }                                                                                                \
  int64_t dpgref_param_count##SFX(const CLayer* layers, int nlayers) {                             \
    RngStream r = RngStream::standard(0);                                                          \
    return static_cast<int64_t>(build_model<T>(descs_of(layers, nlayers), r).parameter_count());   \
  }                                                                                                \
  int dpgref_rule_linear##SFX(const T* acts, const T* hw, int64_t b, int64_t mid, int64_t d,       \
                              int64_t r, T* gw, T* gb) {                                           \
    return guarded([&] {                                                                           \
      Tensor<T> a = tensor_of<T>({(size_t)b, (size_t)mid, (size_t)d}, acts);                       \
      Tensor<T> h = tensor_of<T>({(size_t)b, (size_t)mid, (size_t)r}, hw);                         \
      auto [w, bias] = per_sample_rule_linear(a, h);                                               \
      std::memcpy(gw, w.data(), sizeof(T) * w.numel());                                            \
      if (gb) std::memcpy(gb, bias.data(), sizeof(T) * bias.numel());                              \
    });                                                                                            \
  }                                                                                                \
  int dpgref_rule_conv2d##SFX(const T* x, const T* hw, int64_t b, int64_t ic, int64_t h,           \
                              int64_t w, int64_t oc, int64_t kh, int64_t kw, int64_t stride,       \
                              int64_t pad, T* gw, T* gb) {                                         \
    return guarded([&] {                                                                           \
      LayerDescriptor d = LayerDescriptor::conv2d(ic, oc, kh, kw, stride, pad, true);              \
      LayerCache<T> cache;                                                                         \
      cache.valid = true;                                                                          \
      cache.input = tensor_of<T>({(size_t)b, (size_t)ic, (size_t)h, (size_t)w}, x);                \
      const std::size_t oh = detail::conv_out_extent(h, kh, stride, pad);                          \
      const std::size_t ow = detail::conv_out_extent(w, kw, stride, pad);                          \
      Tensor<T> hwt = tensor_of<T>({(size_t)b, (size_t)oc, oh, ow}, hw);                           \
      auto [gwt, gbt] = per_sample_rule_conv2d(d, cache, hwt);                                     \
      std::memcpy(gw, gwt.data(), sizeof(T) * gwt.numel());                                        \
      if (gb) std::memcpy(gb, gbt.data(), sizeof(T) * gbt.numel());                                \
    });                                                                                            \
  }                                                                                                \
  /* per_sample_rule_layer_norm / _group_norm on [b, q, c] / [b, c, q] with a given cache */    \
  int dpgref_rule_norm##SFX(int group, const T* normalized, const T* hw, int64_t b, int64_t c,     \
                            int64_t q, T* gg, T* gb) {                                             \
    return guarded([&] {                                                                           \
      LayerDescriptor d = group ? LayerDescriptor::group_norm(1, c)                                \
                                : LayerDescriptor::layer_norm(Shape{(std::size_t)c});              \
      const Shape shp = group ? Shape{(size_t)b, (size_t)c, (size_t)q} : Shape{(size_t)b, (size_t)q, (size_t)c}; \
      LayerCache<T> cache;                                                                         \
      cache.valid = true;                                                                          \
      cache.input = Tensor<T>(shp);                                                                \
      cache.normalized = tensor_of<T>(shp, normalized);                                            \
      Tensor<T> h = tensor_of<T>(shp, hw);                                                         \
      auto [g1, g2] = group ? per_sample_rule_group_norm(d, cache, h) : per_sample_rule_layer_norm(d, cache, h); \
      std::memcpy(gg, g1.data(), sizeof(T) * g1.numel());                                          \
      std::memcpy(gb, g2.data(), sizeof(T) * g2.numel());                                          \
    });                                                                                            \
  }                                                                                                \
  int dpgref_rule_embedding##SFX(const T* idx, const T* hw, int64_t b, int64_t t, int64_t vocab,   \
                                 int64_t dim, T* out) {                                            \
    return guarded([&] {                                                                           \
      Tensor<T> it = tensor_of<T>({(size_t)b, (size_t)t}, idx);                                    \
      Tensor<T> ht = tensor_of<T>({(size_t)b, (size_t)t, (size_t)dim}, hw);                        \
      Tensor<T> o = per_sample_rule_embedding(it, ht, vocab);                                      \
      std::memcpy(out, o.data(), sizeof(T) * o.numel());                                           \
    });                                                                                            \
  }                                                                                                \
  int dpgref_clip_and_sum##SFX(const T* const* g, const int64_t* numel, int nparams, int64_t b,    \
                               double c, T* const* summed, double* norms, double* scales,          \
                               int64_t* num_clipped) {                                             \
    return guarded([&] {                                                                           \
      GradSampleRecord<T> rec;                                                                     \
      rec.batch_size = b;                                                                          \
      rec.per_layer.resize(nparams);                                                               \
      rec.param_names.resize(nparams);                                                             \
      for (int p = 0; p < nparams; ++p) {                                                          \
        rec.per_layer[p].push_back(tensor_of<T>({(size_t)b, (size_t)numel[p]}, g[p]));             \
        rec.param_names[p].push_back("p" + std::to_string(p));                                     \
      }                                                                                            \
      auto [s, cs] = clip_and_sum(rec, c);                                                         \
      for (int p = 0; p < nparams; ++p)                                                            \
        std::memcpy(summed[p], s[p][0].data(), sizeof(T) * numel[p]);                              \
      std::memcpy(norms, cs.per_sample_norms.data(), sizeof(double) * b);                          \
      std::memcpy(scales, cs.scale_factors.data(), sizeof(double) * b);                            \
      *num_clipped = static_cast<int64_t>(cs.num_clipped);                                         \
    });                                                                                            \
  }                                                                                                \
  int dpgref_add_noise##SFX(const T* summed, int64_t n, double sigma, double c, uint64_t seed,     \
                            T* out) {                                                              \
    return guarded([&] {                                                                           \
      SummedGrads<T> s(1);                                                                         \
      s[0].push_back(tensor_of<T>({(size_t)n}, summed));                                           \
      RngStream r = RngStream::standard(seed);                                                     \
      SummedGrads<T> o = add_noise(s, sigma, c, r);                                                \
      std::memcpy(out, o[0][0].data(), sizeof(T) * n);                                             \
    });                                                                                            \
  }                                                                                                \
  int dpgref_dpsgd_step##SFX(const CLayer* layers, int nlayers, const int64_t* in_shape,           \
                             int in_rank, int64_t b, const int64_t* shard_sizes, int nshards,      \
                             T* params, const T* x, const T* targets, double sigma, double c,      \
                             double lr, double e, uint64_t seed, const T* injected, T* record,     \
                             T* summed, T* grad, double* norms, double* scales,                    \
                             int64_t* num_clipped, T* loss, T* logits) {                           \
    return guarded([&] {                                                                           \
      dpsgd_step<T>(layers, nlayers, in_shape, in_rank, b, shard_sizes, nshards, params, x,        \
                    targets, sigma, c, lr, e, seed, injected, record, summed, grad, norms, scales, \
                    num_clipped, loss, logits);                                                    \
    });                                                                                            \
  }                                                                                                \
  int dpgref_dpsgd_step_threads##SFX(const CLayer* layers, int nlayers, const int64_t* in_shape,   \
                                     int in_rank, int64_t b, int nthreads, T* params, const T* x,  \
                                     const T* targets, double sigma, double c, double lr,          \
                                     double e, uint64_t seed) {                                    \
    return guarded([&] {                                                                           \
      dpsgd_step_threads<T>(layers, nlayers, in_shape, in_rank, b, nthreads, params, x, targets,   \
                            sigma, c, lr, e, seed);                                                \
    });                                                                                            \
  }                                                                                                \
  int dpgref_microbatch_oracle##SFX(const CLayer* layers, int nlayers, const int64_t* in_shape,    \
                                    int in_rank, int64_t b, const T* params, const T* x,           \
                                    const T* targets, T* record) {                                 \
    return guarded([&] {                                                                           \
      ModelGraph<T> m = model_of<T>(layers, nlayers, params);                                      \
      Shape xs{(size_t)b};                                                                         \
      for (int i = 0; i < in_rank; ++i) xs.push_back((size_t)in_shape[i]);                         \
      std::size_t per = 1;                                                                         \
      for (int i = 0; i < in_rank; ++i) per *= (size_t)in_shape[i];                                \
      Tensor<T> xt = tensor_of<T>(xs, x);                                                          \
      Tensor<T> yt = tensor_of<T>({(size_t)b}, targets);                                           \
      GradSampleRecord<T> rec = microbatch_oracle(m, xt, yt, LossKind::softmax_cross_entropy);     \
      flatten_into(rec.per_layer, record);                                                         \
      (void)per;                                                                                   \
    });                                                                                            \
  }

DPGREF_INSTANTIATE(float, _f32)
DPGREF_INSTANTIATE(double, _f64)

}  // extern "C"
