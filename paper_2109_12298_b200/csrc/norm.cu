// norm.cu — layer_norm and group_norm on the device (SURVEY.md §8f "next" row 2):
//
//   forward        layers.hpp:468-551   xhat = (x - mu) * inv_std, y = gamma * xhat + beta
//   backward_input layers.hpp:650-711   gx = inv (g gamma - mean(g gamma) - xhat mean(g gamma xhat))
//   per-sample     grad_sample.hpp:87-131
//                  ggamma[n][c] = sum_q hw[n, c, q] * xhat[n, c, q],  gbeta[n][c] = sum_q hw[n, c, q]
//                  + their squared norms (the clip pass, optimizer.hpp:67-89)
//
// Both layers are per-row reductions over a few hundred to a few thousand elements, HBM-bound.
// Every reduction runs in the reference's order and precision — one thread owns one row /
// (sample, group) / (sample, channel) and accumulates sequentially (double for the statistics,
// fp32 with separate multiply and add for the rule, as the reference's `acc += a * b` in float
// built without FMA contraction) — so the device results are the reference's bits.
//
// Element addressing: layer_norm over the trailing C features of [b, P, C] (P positions per
// sample): element (n, c, q) = (n P + q) C + c. group_norm over [b, C, S] (S spatial):
// element (n, c, q) = (n C + c) S + q. Both are (n, c, q) -> n*P*C + c*sc + q*sq.
#include "dpg_device.cuh"

namespace dpg {

namespace {

struct NormIdx {
  int64_t per_sample, sc, sq;  // sample stride, channel stride, position stride
  __device__ __forceinline__ int64_t at(int64_t n, int64_t c, int64_t q) const {
    return n * per_sample + c * sc + q * sq;
  }
};

NormIdx ln_idx(int64_t positions, int64_t m) { return NormIdx{positions * m, 1, m}; }
NormIdx gn_idx(int64_t channels, int64_t spatial) { return NormIdx{channels * spatial, spatial, 1}; }

// One thread per statistics block: `cnt_c` channels [c0, c0 + cnt_c) x `cnt_q` positions, walked
// channel-major then position (the reference's loops: layer_norm j over one row; group_norm cg
// then s). Writes xhat, y and inv_std (float, as the reference caches it).
__global__ void norm_fwd_kernel(const float* __restrict__ x, int relu, const float* __restrict__ gamma,
                                const float* __restrict__ beta, NormIdx ix, int64_t b, int64_t blocks_per_sample,
                                int64_t cnt_c, int64_t cnt_q, int gn, double eps, float* __restrict__ y,
                                float* __restrict__ xhat, float* __restrict__ inv_std) {
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b * blocks_per_sample) return;
  const int64_t n = t / blocks_per_sample, blk = t - n * blocks_per_sample;
  // layer_norm: block = position blk (all C channels); group_norm: block = group blk
  const int64_t c0 = gn ? blk * cnt_c : 0, q0 = gn ? 0 : blk;
  auto elem = [&](int64_t c, int64_t q) { return ix.at(n, c0 + c, q0 + q); };
  double mu = 0.0;
  for (int64_t c = 0; c < cnt_c; ++c)
    for (int64_t q = 0; q < cnt_q; ++q) mu += (double)relu_if(x[elem(c, q)], relu);
  const double cnt = (double)(cnt_c * cnt_q);
  mu /= cnt;
  double var = 0.0;
  for (int64_t c = 0; c < cnt_c; ++c)
    for (int64_t q = 0; q < cnt_q; ++q) {
      const double dx = (double)relu_if(x[elem(c, q)], relu) - mu;
      var += dx * dx;
    }
  var /= cnt;
  const double inv = 1.0 / sqrt(var + eps);
  inv_std[t] = (float)inv;
  for (int64_t c = 0; c < cnt_c; ++c) {
    const float gm = gamma[c0 + c], bt = beta[c0 + c];
    for (int64_t q = 0; q < cnt_q; ++q) {
      const int64_t e = elem(c, q);
      const float xh = (float)(((double)relu_if(x[e], relu) - mu) * inv);
      xhat[e] = xh;
      y[e] = __fadd_rn(__fmul_rn(gm, xh), bt);
    }
  }
}

__global__ void norm_dgrad_kernel(const float* __restrict__ gy, const float* __restrict__ gamma,
                                  const float* __restrict__ xhat, const float* __restrict__ inv_std, NormIdx ix,
                                  int64_t b, int64_t blocks_per_sample, int64_t cnt_c, int64_t cnt_q, int gn,
                                  const float* __restrict__ mask, float* __restrict__ gx) {
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b * blocks_per_sample) return;
  const int64_t n = t / blocks_per_sample, blk = t - n * blocks_per_sample;
  const int64_t c0 = gn ? blk * cnt_c : 0, q0 = gn ? 0 : blk;
  auto elem = [&](int64_t c, int64_t q) { return ix.at(n, c0 + c, q0 + q); };
  const double inv = (double)inv_std[t];
  double sum_g = 0.0, sum_gx = 0.0;
  for (int64_t c = 0; c < cnt_c; ++c)
    for (int64_t q = 0; q < cnt_q; ++q) {
      const int64_t e = elem(c, q);
      const double gh = (double)gy[e] * (double)gamma[c0 + c];
      sum_g += gh;
      sum_gx += gh * (double)xhat[e];
    }
  const double cnt = (double)(cnt_c * cnt_q);
  const double mg = sum_g / cnt, mgx = sum_gx / cnt;
  for (int64_t c = 0; c < cnt_c; ++c)
    for (int64_t q = 0; q < cnt_q; ++q) {
      const int64_t e = elem(c, q);
      const double gh = (double)gy[e] * (double)gamma[c0 + c];
      float v = (float)(inv * (gh - mg - (double)xhat[e] * mgx));
      if (mask && !(mask[e] > 0.f)) v = 0.f;  // the producing layer's relu (layers.hpp:712-718)
      gx[e] = v;
    }
}

// One CTA per sample; thread c owns channel c (strided): sequential fp32 sums over the sample's
// positions, then the squared norms of the two records reduced over the CTA in a fixed tree.
__global__ void __launch_bounds__(256) norm_rule_kernel(const float* __restrict__ hw,
                                                        const float* __restrict__ xhat, NormIdx ix,
                                                        int64_t channels, int64_t positions,
                                                        float* __restrict__ gg, float* __restrict__ gb,
                                                        double* __restrict__ sq_g, double* __restrict__ sq_b,
                                                        int64_t b) {
  pdl_wait();
  const int64_t n = blockIdx.x;
  double sg = 0.0, sb = 0.0;
  for (int64_t c = threadIdx.x; c < channels; c += blockDim.x) {
    float ag = 0.f, ab = 0.f;
    for (int64_t q = 0; q < positions; ++q) {
      const int64_t e = ix.at(n, c, q);
      const float h = hw[e];
      ag = __fadd_rn(ag, __fmul_rn(h, xhat[e]));
      ab = __fadd_rn(ab, h);
    }
    if (gg) gg[n * channels + c] = ag;
    if (gb) gb[n * channels + c] = ab;
    sg += (double)ag * ag;
    sb += (double)ab * ab;
  }
  __shared__ double red[2][8];
  const double tg = block_sum<256>(sg, red[0]);
  const double tb = block_sum<256>(sb, red[1]);
  if (threadIdx.x == 0) {
    if (sq_g) sq_g[n] = tg;
    if (sq_b) sq_b[n] = tb;
  }
}

unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_layer_norm_fwd(dpg_ctx* ctx, const float* x, int relu, const float* gamma, const float* beta,
                           int64_t b, int64_t positions, int64_t m, double eps, float* y, float* xhat,
                           float* inv_std) {
  if (b == 0) return;
  ::dpg::launch_pdl(norm_fwd_kernel, blocks_for(b * positions, 128), 128, 0, ctx->stream, 
      x, relu, gamma, beta, ln_idx(positions, m), b, positions, m, 1, 0, eps, y, xhat, inv_std);
  DPG_LAUNCH_CHECK(ctx);
}

void launch_layer_norm_dgrad(dpg_ctx* ctx, const float* gy, const float* gamma, const float* xhat,
                             const float* inv_std, int64_t b, int64_t positions, int64_t m,
                             const float* mask, float* gx) {
  if (b == 0) return;
  ::dpg::launch_pdl(norm_dgrad_kernel, blocks_for(b * positions, 128), 128, 0, ctx->stream, 
      gy, gamma, xhat, inv_std, ln_idx(positions, m), b, positions, m, 1, 0, mask, gx);
  DPG_LAUNCH_CHECK(ctx);
}

void launch_group_norm_fwd(dpg_ctx* ctx, const float* x, int relu, const float* gamma, const float* beta,
                           int64_t b, int64_t channels, int64_t spatial, int64_t groups, double eps,
                           float* y, float* xhat, float* inv_std) {
  if (b == 0) return;
  ::dpg::launch_pdl(norm_fwd_kernel, blocks_for(b * groups, 128), 128, 0, ctx->stream, 
      x, relu, gamma, beta, gn_idx(channels, spatial), b, groups, channels / groups, spatial, 1, eps, y,
      xhat, inv_std);
  DPG_LAUNCH_CHECK(ctx);
}

void launch_group_norm_dgrad(dpg_ctx* ctx, const float* gy, const float* gamma, const float* xhat,
                             const float* inv_std, int64_t b, int64_t channels, int64_t spatial,
                             int64_t groups, const float* mask, float* gx) {
  if (b == 0) return;
  ::dpg::launch_pdl(norm_dgrad_kernel, blocks_for(b * groups, 128), 128, 0, ctx->stream, 
      gy, gamma, xhat, inv_std, gn_idx(channels, spatial), b, groups, channels / groups, spatial, 1, mask, gx);
  DPG_LAUNCH_CHECK(ctx);
}

void launch_norm_rule(dpg_ctx* ctx, const float* hw, const float* xhat, int64_t b, int64_t channels,
                      int64_t positions, bool group_layout, float* gg, float* gb, double* sq_g, double* sq_b) {
  if (b == 0) return;
  const NormIdx ix = group_layout ? gn_idx(channels, positions) : ln_idx(positions, channels);
  ::dpg::launch_pdl(norm_rule_kernel, (unsigned)b, 256, 0, ctx->stream, hw, xhat, ix, channels, positions, gg, gb, sq_g,
                                                         sq_b, b);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace dpg
