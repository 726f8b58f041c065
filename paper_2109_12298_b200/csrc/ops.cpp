// ops.cpp — operator ABI (include/dpg.h, part 1): argument checks with the reference's error
// classes and messages, then the kernel launchers. Asynchronous on the context stream.
#include <string>
#include <vector>

#include "dpg_internal.h"

using dpg::ConvGeom;
using dpg::guard;
using dpg::raise;

namespace {

int64_t conv_out_extent(int64_t in, int64_t kernel, int64_t stride, int64_t pad) {
  // detail::conv_out_extent (layers.hpp:283-288)
  const int64_t padded = in + 2 * pad;
  if (padded < kernel) return 0;
  return (padded - kernel) / stride + 1;
}

ConvGeom conv_geom(int64_t b, int64_t h, int64_t w, const dpg_conv2d_spec* s) {
  if (!s) raise(DPG_ERR_PARAMETER, "conv2d: null spec");
  if (s->in_channels <= 0 || s->out_channels <= 0 || s->kernel_h <= 0 || s->kernel_w <= 0 ||
      s->stride <= 0 || s->padding < 0)
    raise(DPG_ERR_PARAMETER, "conv2d: channel, kernel, and stride extents must be positive");
  ConvGeom g{b, s->in_channels, h, w, s->out_channels, s->kernel_h, s->kernel_w, s->stride,
             s->padding, conv_out_extent(h, s->kernel_h, s->stride, s->padding),
             conv_out_extent(w, s->kernel_w, s->stride, s->padding)};
  if (g.oh == 0 || g.ow == 0) raise(DPG_ERR_DIMENSION, "conv2d: kernel larger than padded input");
  return g;
}

void need(const void* p, const char* what) {
  if (!p) raise(DPG_ERR_PARAMETER, std::string(what) + " must not be NULL");
}

void need_ctx(dpg_ctx* ctx) {
  if (!ctx) raise(DPG_ERR_PARAMETER, "null context");
  DPG_CUDA(cudaSetDevice(ctx->device));
}

// Workspace each operator takes from the context arena (the dpg_*_workspace_size queries return
// these, so a caller can dpg_ctx_reserve_workspace once and no hot call allocates).
size_t ws_gs_linear(int64_t b, int64_t mid, int64_t d, int64_t r) {
  return sizeof(double) * (size_t)dpg::sq_rows_linear(mid, d, r) * (size_t)b;
}
size_t ws_gs_conv2d(const ConvGeom& g) { return sizeof(double) * (size_t)dpg::sq_rows_conv2d(g) * (size_t)g.b; }
size_t ws_embed_sort(int64_t b, int64_t t) { return sizeof(int32_t) * 2 * (size_t)(b * t); }
size_t ws_gs_embedding(int64_t b, int64_t t, int64_t vocab, int64_t dim) {
  return ws_embed_sort(b, t) + sizeof(double) * (size_t)dpg::sq_rows_embedding(vocab, dim) * (size_t)b;
}
size_t ws_cs_linear(int64_t b, int64_t mid, int64_t d, int64_t r) {
  return dpg::clipped_sum_ws_linear(b, mid, d, r) + sizeof(float) * (size_t)(b * r);
}
size_t ws_cs_conv2d(const ConvGeom& g) { return dpg::clipped_sum_ws_conv2d(g) + sizeof(float) * (size_t)(g.b * g.oc); }
size_t ws_cs_embedding(int64_t b, int64_t t, int64_t vocab) {
  return ws_embed_sort(b, t) + dpg::clipped_sum_ws_embedding(b, vocab);
}

// a query never raises: invalid extents report 0
template <class F>
size_t ws_query(F&& f) {
  try {
    return f();
  } catch (...) {
    return 0;
  }
}

}  // namespace

extern "C" {

dpg_status dpg_grad_sample_linear(dpg_ctx* ctx, const float* acts, const float* highway, int64_t b,
                                  int64_t mid, int64_t d, int64_t r, float* gw, float* gb,
                                  double* sq_w, double* sq_b) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(acts, "acts");
    need(highway, "highway");
    if (b < 0 || mid <= 0 || d <= 0 || r <= 0)
      raise(DPG_ERR_DIMENSION, "batched_outer: extents must be positive");
    if (b == 0) return;
    const int rows = dpg::sq_rows_linear(mid, d, r);
    double* part = sq_w ? static_cast<double*>(ctx->workspace(ws_gs_linear(b, mid, d, r))) : nullptr;
    // T > 1: the bias rule (a pass over the whole highway) runs on the side stream beside the
    // weight rule; the call is joined before it returns
    const bool side = (gb || sq_b) && mid > 1 && ctx->can_fork();
    if (side) {
      ctx->fork_side();
      dpg::launch_gs_bias(ctx, highway, b, mid, r, false, gb, sq_b);
      ctx->end_side();
    }
    dpg::launch_gs_linear(ctx, acts, 0, highway, b, mid, d, r, gw, part);
    if (sq_w) dpg::launch_sq_reduce(ctx, part, rows, b, sq_w);
    if (side) ctx->join_side();
    else if (gb || sq_b) dpg::launch_gs_bias(ctx, highway, b, mid, r, false, gb, sq_b);
  });
}

dpg_status dpg_grad_sample_conv2d(dpg_ctx* ctx, const float* x, const float* highway, int64_t b,
                                  int64_t h, int64_t w, const dpg_conv2d_spec* spec, float* gw,
                                  float* gb, double* sq_w, double* sq_b) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(x, "x");
    need(highway, "highway");
    const ConvGeom g = conv_geom(b, h, w, spec);
    if (b == 0) return;
    const int rows = dpg::sq_rows_conv2d(g);
    double* part = sq_w ? static_cast<double*>(ctx->workspace(ws_gs_conv2d(g))) : nullptr;
    dpg::launch_gs_conv2d(ctx, x, 0, highway, g, gw, part);
    if (sq_w) dpg::launch_sq_reduce(ctx, part, rows, b, sq_w);
    if (gb || sq_b) dpg::launch_gs_bias(ctx, highway, b, g.P(), g.oc, true, gb, sq_b);
  });
}

static dpg_status norm_rule(dpg_ctx* ctx, const float* normalized, const float* highway, int64_t b,
                            int64_t channels, int64_t positions, bool group_layout, float* gg, float* gb,
                            double* sq_g, double* sq_b, const char* who) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(normalized, "normalized");
    need(highway, "highway");
    if (b < 0 || channels <= 0 || positions <= 0)
      raise(DPG_ERR_DIMENSION, std::string(who) + ": extents must be positive");
    if (b == 0) return;
    dpg::launch_norm_rule(ctx, highway, normalized, b, channels, positions, group_layout, gg, gb, sq_g, sq_b);
  });
}

dpg_status dpg_grad_sample_layer_norm(dpg_ctx* ctx, const float* normalized, const float* highway, int64_t b,
                                      int64_t positions, int64_t m, float* ggamma, float* gbeta,
                                      double* sq_gamma, double* sq_beta) {
  return norm_rule(ctx, normalized, highway, b, m, positions, false, ggamma, gbeta, sq_gamma, sq_beta,
                   "layer_norm");
}

dpg_status dpg_grad_sample_group_norm(dpg_ctx* ctx, const float* normalized, const float* highway, int64_t b,
                                      int64_t channels, int64_t spatial, float* ggamma, float* gbeta,
                                      double* sq_gamma, double* sq_beta) {
  return norm_rule(ctx, normalized, highway, b, channels, spatial, true, ggamma, gbeta, sq_gamma, sq_beta,
                   "group_norm");
}

dpg_status dpg_grad_sample_embedding(dpg_ctx* ctx, const float* idx, const float* highway,
                                     int64_t b, int64_t t, int64_t vocab, int64_t dim, float* g,
                                     double* sq) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(idx, "idx");
    need(highway, "highway");
    if (vocab <= 0 || dim <= 0) raise(DPG_ERR_PARAMETER, "embedding: extents must be positive");
    if (b == 0 || t == 0) return;
    const int rows = dpg::sq_rows_embedding(vocab, dim);
    const size_t sort_bytes = ws_embed_sort(b, t);
    char* ws = static_cast<char*>(ctx->workspace(ws_gs_embedding(b, t, vocab, dim)));
    int32_t* sv = reinterpret_cast<int32_t*>(ws);
    int32_t* ss = sv + b * t;
    double* part = reinterpret_cast<double*>(ws + sort_bytes);
    dpg::launch_embed_sort(ctx, idx, b, t, vocab, sv, ss);
    dpg::launch_gs_embedding(ctx, sv, ss, highway, b, t, vocab, dim, g, part);
    if (sq) dpg::launch_sq_reduce(ctx, part, rows, b, sq);
  });
}

dpg_status dpg_clip_factors(dpg_ctx* ctx, const double* sq, int nparams, int64_t b, double c,
                            double* norms, float* scale, int64_t* num_clipped) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    // optimizer.hpp:64-65
    if (!(c > 0.0)) raise(DPG_ERR_PARAMETER, "clipping threshold must be > 0");
    if (b == 0) raise(DPG_ERR_PARAMETER, "clip_and_sum on an empty batch");
    need(sq, "sq");
    need(scale, "scale");
    // row r of the slab is parameter r: a device-resident identity map (no host copy, no sync)
    const int32_t* drp = ctx->identity_rows(nparams > 0 ? nparams : 1);
    dpg::launch_clip_factors(ctx, sq, drp, nparams, b, c, norms, scale, num_clipped);
  });
}

dpg_status dpg_clipped_sum_linear(dpg_ctx* ctx, const float* acts, const float* highway,
                                  const float* scale, int64_t b, int64_t mid, int64_t d, int64_t r,
                                  float* sw, float* sb, int accumulate) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(acts, "acts");
    need(highway, "highway");
    need(scale, "scale");
    need(sw, "sw");
    if (b <= 0) raise(DPG_ERR_PARAMETER, "clip_and_sum on an empty batch");
    void* ws = ctx->workspace(ws_cs_linear(b, mid, d, r));
    // bias: weighted sum of the per-sample bias sums (bit-exact with the reference); T > 1: on the
    // side stream, beside the weight's clipped sum (its own slice of the workspace)
    const bool side = sb && mid > 1 && ctx->can_fork();
    float* gb = sb ? reinterpret_cast<float*>(static_cast<char*>(ws) + dpg::clipped_sum_ws_linear(b, mid, d, r)) : nullptr;
    if (side) {
      ctx->fork_side();
      dpg::launch_gs_bias(ctx, highway, b, mid, r, false, gb, nullptr);
      dpg::launch_weighted_sum_materialised(ctx, gb, scale, b, r, sb, accumulate);
      ctx->end_side();
    }
    dpg::launch_clipped_sum_linear(ctx, acts, 0, highway, scale, b, mid, d, r, sw, sb, accumulate, ws);
    if (side) {
      ctx->join_side();
    } else if (sb) {
      dpg::launch_gs_bias(ctx, highway, b, mid, r, false, gb, nullptr);
      dpg::launch_weighted_sum_materialised(ctx, gb, scale, b, r, sb, accumulate);
    }
  });
}

dpg_status dpg_clipped_sum_conv2d(dpg_ctx* ctx, const float* x, const float* highway,
                                  const float* scale, int64_t b, int64_t h, int64_t w,
                                  const dpg_conv2d_spec* spec, float* sw, float* sb,
                                  int accumulate) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(x, "x");
    need(highway, "highway");
    need(scale, "scale");
    need(sw, "sw");
    const ConvGeom g = conv_geom(b, h, w, spec);
    if (b <= 0) raise(DPG_ERR_PARAMETER, "clip_and_sum on an empty batch");
    const size_t wsz = dpg::clipped_sum_ws_conv2d(g);
    void* ws = ctx->workspace(ws_cs_conv2d(g));
    dpg::launch_clipped_sum_conv2d(ctx, x, 0, highway, scale, g, sw, sb, accumulate, ws);
    if (sb) {
      float* gb = reinterpret_cast<float*>(static_cast<char*>(ws) + wsz);
      dpg::launch_gs_bias(ctx, highway, b, g.P(), g.oc, true, gb, nullptr);
      dpg::launch_weighted_sum_materialised(ctx, gb, scale, b, g.oc, sb, accumulate);
    }
  });
}

dpg_status dpg_clipped_sum_embedding(dpg_ctx* ctx, const float* idx, const float* highway,
                                     const float* scale, int64_t b, int64_t t, int64_t vocab,
                                     int64_t dim, float* summed, int accumulate) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(idx, "idx");
    need(highway, "highway");
    need(scale, "scale");
    need(summed, "summed");
    if (b <= 0) raise(DPG_ERR_PARAMETER, "clip_and_sum on an empty batch");
    const size_t sort_bytes = ws_embed_sort(b, t);
    char* ws = static_cast<char*>(ctx->workspace(ws_cs_embedding(b, t, vocab)));
    int32_t* sv = reinterpret_cast<int32_t*>(ws);
    int32_t* ss = sv + b * t;
    dpg::launch_embed_sort(ctx, idx, b, t, vocab, sv, ss);
    dpg::launch_clipped_sum_embedding(ctx, sv, ss, highway, scale, b, t, vocab, dim, summed,
                                      accumulate, ws + sort_bytes);
  });
}

dpg_status dpg_clip_and_sum_materialised(dpg_ctx* ctx, const float* const* g, const int64_t* numel,
                                         int nparams, int64_t b, double c, float* const* summed,
                                         double* norms, float* scale, int64_t* num_clipped,
                                         int accumulate) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    if (!(c > 0.0)) raise(DPG_ERR_PARAMETER, "clipping threshold must be > 0");
    if (b == 0) raise(DPG_ERR_PARAMETER, "clip_and_sum on an empty batch");
    need(scale, "scale");
    std::vector<int32_t> rp;
    std::vector<int> row0(nparams);
    for (int p = 0; p < nparams; ++p) {
      row0[p] = (int)rp.size();
      const int rows = dpg::sq_rows_materialised(numel[p]);
      for (int r = 0; r < rows; ++r) rp.push_back(p);
    }
    const int rows = (int)rp.size();
    char* ws = static_cast<char*>(ctx->workspace(sizeof(double) * rows * b + sizeof(int32_t) * (rows + 1)));
    double* slab = reinterpret_cast<double*>(ws);
    int32_t* drp = reinterpret_cast<int32_t*>(ws + sizeof(double) * rows * b);
    if (rows > 0)
      DPG_CUDA(cudaMemcpyAsync(drp, rp.data(), sizeof(int32_t) * rows, cudaMemcpyHostToDevice, ctx->stream));
    for (int p = 0; p < nparams; ++p) dpg::launch_sq_materialised(ctx, g[p], b, numel[p], slab + (int64_t)row0[p] * b);
    dpg::launch_clip_factors(ctx, slab, drp, rows, b, c, norms, scale, num_clipped);
    for (int p = 0; p < nparams; ++p)
      dpg::launch_weighted_sum_materialised(ctx, g[p], scale, b, numel[p], summed[p], accumulate);
    DPG_CUDA(cudaStreamSynchronize(ctx->stream));  // rp is a host temporary
  });
}

dpg_status dpg_noise_update(dpg_ctx* ctx, float* params, const float* summed, float* grad,
                            int64_t n, double sigma, double c, double expected_batch, double lr,
                            uint64_t seed, uint64_t step, const float* injected_noise) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(params, "params");
    need(summed, "summed");
    if (sigma < 0.0) raise(DPG_ERR_PARAMETER, "noise multiplier must be >= 0");
    if (!(c > 0.0)) raise(DPG_ERR_PARAMETER, "max grad norm must be > 0");
    if (!(lr > 0.0)) raise(DPG_ERR_PARAMETER, "learning rate must be > 0");
    if (!(expected_batch > 0.0)) raise(DPG_ERR_PARAMETER, "expected batch size must be > 0");
    dpg::launch_noise_update(ctx, params, summed, grad, n, sigma, c, expected_batch, lr, seed, step,
                             injected_noise, nullptr);
  });
}

dpg_status dpg_gaussian(dpg_ctx* ctx, float* out, int64_t n, double std_dev, uint64_t seed,
                        uint64_t step) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    need(out, "out");
    if (std_dev < 0.0) raise(DPG_ERR_PARAMETER, "gaussian: std must be non-negative");
    dpg::launch_gaussian(ctx, out, n, std_dev, seed, step);
  });
}


size_t dpg_grad_sample_linear_workspace_size(int64_t b, int64_t mid, int64_t d, int64_t r) {
  return ws_query([&] { return (b > 0 && mid > 0 && d > 0 && r > 0) ? ws_gs_linear(b, mid, d, r) : size_t(0); });
}
size_t dpg_grad_sample_conv2d_workspace_size(int64_t b, int64_t h, int64_t w, const dpg_conv2d_spec* spec) {
  return ws_query([&] { return b > 0 ? ws_gs_conv2d(conv_geom(b, h, w, spec)) : size_t(0); });
}
size_t dpg_grad_sample_embedding_workspace_size(int64_t b, int64_t t, int64_t vocab, int64_t dim) {
  return ws_query([&] { return (b > 0 && t > 0 && vocab > 0 && dim > 0) ? ws_gs_embedding(b, t, vocab, dim) : size_t(0); });
}
size_t dpg_clipped_sum_linear_workspace_size(int64_t b, int64_t mid, int64_t d, int64_t r) {
  return ws_query([&] { return (b > 0 && mid > 0 && d > 0 && r > 0) ? ws_cs_linear(b, mid, d, r) : size_t(0); });
}
size_t dpg_clipped_sum_conv2d_workspace_size(int64_t b, int64_t h, int64_t w, const dpg_conv2d_spec* spec) {
  return ws_query([&] { return b > 0 ? ws_cs_conv2d(conv_geom(b, h, w, spec)) : size_t(0); });
}
size_t dpg_clipped_sum_embedding_workspace_size(int64_t b, int64_t t, int64_t vocab, int64_t dim) {
  return ws_query([&] { return (b > 0 && t > 0 && vocab > 0 && dim > 0) ? ws_cs_embedding(b, t, vocab) : size_t(0); });
}

dpg_status dpg_ctx_reserve_workspace(dpg_ctx* ctx, size_t bytes) {
  return guard(ctx, [&] {
    need_ctx(ctx);
    ctx->workspace(bytes);
  });
}
}  // extern "C"
