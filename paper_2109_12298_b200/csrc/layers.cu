// layers.cu — supporting forward / input-backward kernels for the full step on the device
// (SURVEY.md §8a rows a12-a14): conv2d forward (implicit GEMM) and dgrad, linear forward and
// dgrad, embedding gather, softmax cross-entropy. ReLU layers are folded into their consumers:
// activations are stored pre-ReLU and the ReLU is applied on load (forward) or as a mask in
// the producing dgrad epilogue (backward, layers.hpp:712-718).
#include "conv_common.cuh"
#include "step_common.cuh"
#include "igemm.cuh"

namespace dpg {

// ------------------------------------------------------------------------------------------
// conv2d forward (layers.hpp:432-467) and dgrad (:630-649): tcgen05 implicit GEMMs (tc_conv.cu);
// a SIMT gather-form dgrad remains for geometries the tcgen05 tap tables do not cover
// (stride > 4, output extents >= 255).
// ------------------------------------------------------------------------------------------
size_t conv_fwd_ws_bytes(const ConvGeom& g) {
  return tc::fwd_ws_bytes(g);
}
size_t conv_dgrad_ws_bytes(const ConvGeom& g) {
  return tc::dgrad_supported(g) ? tc::dgrad_ws_bytes(g) : 0;
}

// Thin first layers (K = ic kh kw <= KMAX, e.g. an RGB or greyscale image) on the CUDA cores: the
// contraction is 27-64 deep, so a tensor-core tile would be mostly padding and the launch is
// bound by its stores. Thread = output pixel: its K input values (zero padding, ReLU on load)
// in registers, the transposed weights [k][oc] and the bias in shared memory (broadcast float4
// reads), OC fp32 accumulators (bias first, then k ascending — layers.hpp:432-467's sum
// order per output), then the NCHW output (one coalesced store per channel) and the consumer's
// NHWC copy (OC contiguous floats per pixel, ReLU applied when relu_out).
template <int OC, int IC, int KH, int KW>
__global__ void __launch_bounds__(256) conv_fwd_thin_kernel(const float* __restrict__ x, int x_relu,
                                                            const float* __restrict__ w,
                                                            const float* __restrict__ bias, ConvGeom g,
                                                            float* __restrict__ y, float* __restrict__ yh,
                                                            int relu_out) {
  constexpr int K = IC * KH * KW;
  __shared__ __align__(16) float wt[K][OC];
  __shared__ __align__(16) float bs[OC];
  pdl_wait();
  for (int i = threadIdx.x; i < OC * K; i += blockDim.x) {
    const int o = i / K, k = i - o * K;
    wt[k][o] = __ldg(w + i);
  }
  for (int i = threadIdx.x; i < OC; i += blockDim.x) bs[i] = bias ? __ldg(bias + i) : 0.f;
  __syncthreads();
  const int P = (int)(g.oh * g.ow), pblocks = (P + 255) / 256;
  const int items = (int)g.b * pblocks;
  // persistent: the weights are staged once per CTA, then (sample, 256-pixel block) items
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
  const int n = it / pblocks, p = (it - n * pblocks) * 256 + threadIdx.x;
  if (p >= P) continue;
  const int oy = p / (int)g.ow, ox = p - oy * (int)g.ow;
  const int H = (int)g.h, W = (int)g.w;
  const int iy0 = oy * (int)g.stride - (int)g.pad, ix0 = ox * (int)g.stride - (int)g.pad;
  const float* xn = x + (int64_t)n * IC * H * W;
  float in[K];
#pragma unroll
  for (int c = 0; c < IC; ++c)
#pragma unroll
    for (int ki = 0; ki < KH; ++ki)
#pragma unroll
      for (int kj = 0; kj < KW; ++kj) {
        const int iy = iy0 + ki, ix = ix0 + kj;
        const bool ok = iy >= 0 && iy < H && ix >= 0 && ix < W;
        const float v = ok ? __ldg(xn + ((int64_t)c * H + iy) * W + ix) : 0.f;
        in[(c * KH + ki) * KW + kj] = x_relu ? fmaxf(v, 0.f) : v;
      }
  float acc[OC];
#pragma unroll
  for (int o = 0; o < OC; o += 4) {
    const float4 b4 = *reinterpret_cast<const float4*>(&bs[o]);
    acc[o] = b4.x; acc[o + 1] = b4.y; acc[o + 2] = b4.z; acc[o + 3] = b4.w;
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int o = 0; o < OC; o += 4) {
      const float4 w4 = *reinterpret_cast<const float4*>(&wt[k][o]);
      acc[o] = fmaf(in[k], w4.x, acc[o]);
      acc[o + 1] = fmaf(in[k], w4.y, acc[o + 1]);
      acc[o + 2] = fmaf(in[k], w4.z, acc[o + 2]);
      acc[o + 3] = fmaf(in[k], w4.w, acc[o + 3]);
    }
  float* yn = y + (int64_t)n * OC * P + p;
#pragma unroll
  for (int o = 0; o < OC; ++o) yn[(int64_t)o * P] = acc[o];
  if (yh) {
    float4* hp = reinterpret_cast<float4*>(yh + ((int64_t)n * P + p) * OC);
#pragma unroll
    for (int o = 0; o < OC; o += 4)
      hp[o / 4] = make_float4(relu_if(acc[o], relu_out), relu_if(acc[o + 1], relu_out),
                              relu_if(acc[o + 2], relu_out), relu_if(acc[o + 3], relu_out));
  }
  }
}

template <int OC, int IC, int KH, int KW>
static void launch_fwd_thin(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
                            const ConvGeom& g, float* y, float* yh, int relu_out) {
  const int64_t items = g.b * ((g.P() + 255) / 256);
  const unsigned grid = (unsigned)std::min<int64_t>(items, 2 * kNumSMs);
  ::dpg::launch_pdl(conv_fwd_thin_kernel<OC, IC, KH, KW>, dim3(grid), 256, 0, ctx->stream, x, x_relu, w, bias, g,
                    y, yh, relu_out);
  DPG_LAUNCH_CHECK(ctx);
}

void launch_conv2d_fwd(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
                       const ConvGeom& g, float* y, void* ws, float* yh, int relu_out) {
  if (g.b == 0) return;
  if (g.b < 65536 && g.P() < (1 << 30)) {
    if (g.oc == 32 && g.ic == 3 && g.kh == 3 && g.kw == 3)
      return launch_fwd_thin<32, 3, 3, 3>(ctx, x, x_relu, w, bias, g, y, yh, relu_out);
    if (g.oc == 16 && g.ic == 1 && g.kh == 8 && g.kw == 8)
      return launch_fwd_thin<16, 1, 8, 8>(ctx, x, x_relu, w, bias, g, y, yh, relu_out);
  }
  tc::conv_fwd(ctx, x, x_relu, w, bias, g, y, ws, yh, relu_out);
}

// ------------------------------------------------------------------------------------------
// conv2d dgrad (layers.hpp:630-649 + col2im :326-358), implicit and gather-form: for stride s,
// input pixels split into s*s parity classes (ry, rx) = ((iy+pad) % s, (ix+pad) % s); inside a
// class the valid taps are ki = ry + s*a, kj = rx + s*c, so each class is a dense GEMM
// M = ic, N = b * (class pixels), K = oc * taps with no wasted multiply-adds. The epilogue
// applies the ReLU mask of the previous layer (the relu layer's backward, layers.hpp:712-718).
// ------------------------------------------------------------------------------------------
struct ConvDgradProb {
  static constexpr bool kAMajorM = false;
  static constexpr bool kBMajorN = true;
  static constexpr bool kExact = false;
  const float* dy;
  const float* w;
  const float* mask;
  float* dx;
  int64_t M, N, K;  // M = ic, N = b * hc * wc, K = oc * nki * nkj
  int ic, h, wdt, oc, kh, kw, stride, pad, oh, ow;
  int ry, rx, hc, wc, nki, nkj, iy0, ix0;
  __device__ float init(int, int64_t, int64_t) const { return 0.f; }
  // k = (o * nki + a) * nkj + c  ->  tap (ki, kj) = (ry + s*a, rx + s*c)
  __device__ float a(int, int64_t m, int64_t k) const {
    const int taps = nki * nkj;
    const int o = (int)(k / taps), t = (int)(k - (int64_t)o * taps);
    const int aa = t / nkj, cc = t - aa * nkj;
    const int ki = ry + stride * aa, kj = rx + stride * cc;
    return __ldg(w + (((int64_t)o * ic + m) * kh + ki) * kw + kj);
  }
  __device__ float b(int, int64_t k, int64_t nn) const {
    const int taps = nki * nkj;
    const int o = (int)(k / taps), t = (int)(k - (int64_t)o * taps);
    const int aa = t / nkj, cc = t - aa * nkj;
    const int64_t per = (int64_t)hc * wc;
    const int64_t n = nn / per;
    const int q = (int)(nn - n * per);
    const int qy = q / wc, qx = q - qy * wc;
    const int iy = iy0 + stride * qy, ix = ix0 + stride * qx;
    // oy * s + ki - pad = iy  ->  oy = (iy + pad - ki) / s (exact by construction of the class)
    const int oy = (iy + pad - (ry + stride * aa)) / stride;
    const int ox = (ix + pad - (rx + stride * cc)) / stride;
    if (oy < 0 || oy >= oh || ox < 0 || ox >= ow) return 0.f;
    return __ldg(dy + (((int64_t)n * oc + o) * oh + oy) * ow + ox);
  }
  template <int TM, int TN>
  __device__ void epilogue(int, int64_t m0, int64_t n0, int tx, int ty, float (&acc)[TM][TN]) const {
    const int64_t per = (int64_t)hc * wc;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t m = m0 + ty + 16 * i, nn = n0 + tx + 16 * j;
        if (m < M && nn < N) {
          const int64_t n = nn / per;
          const int q = (int)(nn - n * per);
          const int qy = q / wc, qx = q - qy * wc;
          const int iy = iy0 + stride * qy, ix = ix0 + stride * qx;
          const int64_t off = ((n * ic + m) * h + iy) * (int64_t)wdt + ix;
          float v = acc[i][j];
          if (mask && !(__ldg(mask + off) > 0.f)) v = 0.f;
          dx[off] = v;
        }
      }
  }
};

void launch_conv2d_dgrad(dpg_ctx* ctx, const float* dy, const float* w, const ConvGeom& g,
                         const float* mask_src, float* dx, void* ws) {
  if (g.b == 0) return;
  if (tc::dgrad_supported(g)) {
    tc::conv_dgrad(ctx, dy, w, g, mask_src, dx, ws);
    return;
  }
  const int s = (int)g.stride;
  for (int ry = 0; ry < s; ++ry)
    for (int rx = 0; rx < s; ++rx) {
      ConvDgradProb p{};
      p.dy = dy;
      p.w = w;
      p.mask = mask_src;
      p.dx = dx;
      p.ic = (int)g.ic; p.h = (int)g.h; p.wdt = (int)g.w; p.oc = (int)g.oc;
      p.kh = (int)g.kh; p.kw = (int)g.kw; p.stride = s; p.pad = (int)g.pad;
      p.oh = (int)g.oh; p.ow = (int)g.ow;
      p.ry = ry; p.rx = rx;
      // first input row iy >= 0 with (iy + pad) % s == ry
      p.iy0 = ((ry - (int)g.pad) % s + s) % s;
      p.ix0 = ((rx - (int)g.pad) % s + s) % s;
      p.hc = p.iy0 < g.h ? (int)((g.h - p.iy0 + s - 1) / s) : 0;
      p.wc = p.ix0 < g.w ? (int)((g.w - p.ix0 + s - 1) / s) : 0;
      p.nki = ry < g.kh ? (int)((g.kh - ry + s - 1) / s) : 0;
      p.nkj = rx < g.kw ? (int)((g.kw - rx + s - 1) / s) : 0;
      if (p.hc == 0 || p.wc == 0) continue;
      p.M = g.ic;
      p.N = g.b * p.hc * p.wc;
      p.K = g.oc * p.nki * p.nkj;
      if (p.K == 0) {
        // no tap reaches this class: the input gradient is exactly zero there
        // (handled by a K = 0 GEMM: the epilogue stores the zero accumulators)
      }
      if (g.ic <= 32) launch_igemm<32, 128, 16>(ctx, p, 1);
      else launch_igemm<64, 64, 16>(ctx, p, 1);
    }
}

// ------------------------------------------------------------------------------------------
// linear forward (layers.hpp:389-413): y[r, o] = bias[o] + sum_j W[o, j] x[r, j].
// Narrow outputs (o <= 32, every model on the hot path): one warp per row keeps all o partial
// dot products in registers and reads the row once. Wide outputs: tiled GEMM.
// ------------------------------------------------------------------------------------------
template <int RMAX>
__global__ void __launch_bounds__(256) linear_fwd_narrow_kernel(const float* __restrict__ x,
                                                                int x_relu,
                                                                const float* __restrict__ w,
                                                                const float* __restrict__ bias,
                                                                int64_t rows, int64_t d, int r,
                                                                float* __restrict__ y) {
  pdl_wait();
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float acc[RMAX];
#pragma unroll
  for (int o = 0; o < RMAX; ++o) acc[o] = 0.f;
  const float* xr = x + row * d;
  for (int64_t j = lane; j < d; j += 32) {
    const float xv = relu_if(__ldg(xr + j), x_relu);
#pragma unroll
    for (int o = 0; o < RMAX; ++o)
      if (o < r) acc[o] = fmaf(__ldg(w + (int64_t)o * d + j), xv, acc[o]);
  }
#pragma unroll
  for (int o = 0; o < RMAX; ++o) {
    if (o < r) {
      const float s = warp_sum(acc[o]);
      if (lane == 0) y[row * r + o] = (bias ? __ldg(bias + o) : 0.f) + s;
    }
  }
}

// Narrow outputs (r <= 64) with d % 4 == 0: one CTA per row, its 4 warps split the row's 16-byte
// chunks; every lane keeps the r weight chunks of its column in flight (coalesced 128-bit loads),
// per-row dot products are reduced warp (fixed shuffle tree) then across the 4 warps in order.
template <int RMAX, int NW>  // NW warps per row: 8 for long rows (e.g. 32768 features), else 4
__global__ void __launch_bounds__(32 * NW) linear_fwd_row_kernel(const float* __restrict__ x,
                                                                       int x_relu,
                                                                       const float* __restrict__ w,
                                                                       const float* __restrict__ bias,
                                                                       int64_t d, int r,
                                                                       float* __restrict__ y, LossFuse ce) {
  pdl_wait();
  __shared__ float part[NW][RMAX];
  __shared__ float logit[RMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = blockIdx.x;
  float acc[RMAX];
#pragma unroll
  for (int o = 0; o < RMAX; ++o) acc[o] = 0.f;
  const float4* xr = reinterpret_cast<const float4*>(x + row * d);
  const int64_t d4 = d >> 2;
#pragma unroll 4
  for (int64_t c = (int64_t)warp * 32 + lane; c < d4; c += 32 * NW) {
    float4 xv = __ldg(xr + c);
    xv = make_float4(relu_if(xv.x, x_relu), relu_if(xv.y, x_relu), relu_if(xv.z, x_relu), relu_if(xv.w, x_relu));
#pragma unroll
    for (int o = 0; o < RMAX; ++o) {
      if (o < r) {
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (int64_t)o * d) + c);
        acc[o] = fmaf(wv.x, xv.x, acc[o]);
        acc[o] = fmaf(wv.y, xv.y, acc[o]);
        acc[o] = fmaf(wv.z, xv.z, acc[o]);
        acc[o] = fmaf(wv.w, xv.w, acc[o]);
      }
    }
  }
#pragma unroll
  for (int o = 0; o < RMAX; ++o) {
    if (o < r) {
      const float v = warp_sum(acc[o]);
      if (lane == 0) part[warp][o] = v;
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < r; o += 32 * NW) {
    float t = part[0][o];
#pragma unroll
    for (int q = 1; q < NW; ++q) t += part[q][o];
    const float v = (bias ? __ldg(bias + o) : 0.f) + t;
    y[row * r + o] = v;
    logit[o] = v;
  }
  if (ce.grad) {  // this layer's outputs are the logits: the loss in the same launch
    __syncthreads();
    if (warp == 0) softmax_ce_warp(logit, ce.logits_relu, ce.targets, row, r, ce.loss, ce.grad, ce.err);
    if (ce.dx) {  // and the input gradient: linear_dgrad_vec_kernel's arithmetic, in its order
      __syncthreads();
      __shared__ float g[RMAX];
      if (threadIdx.x < r) g[threadIdx.x] = ce.grad[row * r + threadIdx.x];
      __syncthreads();
      for (int64_t c = threadIdx.x; c < d4; c += 32 * NW) {
        const int64_t j = 4 * c;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int o = 0; o < RMAX; ++o) {
          if (o >= r) break;
          const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (int64_t)o * d + j));
          a.x = fmaf(g[o], wv.x, a.x);
          a.y = fmaf(g[o], wv.y, a.y);
          a.z = fmaf(g[o], wv.z, a.z);
          a.w = fmaf(g[o], wv.w, a.w);
        }
        if (ce.dmask) {
          const float4 mv = __ldg(reinterpret_cast<const float4*>(ce.dmask + row * d + j));
          if (!(mv.x > 0.f)) a.x = 0.f;
          if (!(mv.y > 0.f)) a.y = 0.f;
          if (!(mv.z > 0.f)) a.z = 0.f;
          if (!(mv.w > 0.f)) a.w = 0.f;
        }
        *reinterpret_cast<float4*>(ce.dx + row * d + j) = a;
        if (ce.dx_nhwc) {
          const float e[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int jj = (int)j + u, c = jj / ce.nhwc_p, pp = jj - c * ce.nhwc_p;
            ce.dx_nhwc[row * d + (int64_t)pp * ce.nhwc_c + c] = e[u];
          }
        }
      }
    }
  }
}

// Narrow outputs with d % 4 == 0: a CTA owns kFwdRows rows; thread t walks the 16-byte column
// chunks t, t + 128, ... of those rows, reading each weight chunk once for all of them, so every
// load is a coalesced 128-bit load and each thread keeps ~kFwdRows + 1 of them in flight.
// Per-row dot products are reduced warp then CTA in a fixed order.
constexpr int kFwdRows = 4;
constexpr int kFwdThreads = 128;
template <int RMAX>
__global__ void __launch_bounds__(kFwdThreads) linear_fwd_rows_kernel(const float* __restrict__ x,
                                                                     int x_relu,
                                                                     const float* __restrict__ w,
                                                                     const float* __restrict__ bias,
                                                                     int64_t rows, int64_t d, int r,
                                                                     float* __restrict__ y) {
  pdl_wait();
  __shared__ float red[kFwdThreads / 32][kFwdRows * RMAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * kFwdRows;
  float acc[kFwdRows][RMAX];
#pragma unroll
  for (int i = 0; i < kFwdRows; ++i)
#pragma unroll
    for (int o = 0; o < RMAX; ++o) acc[i][o] = 0.f;
  const int64_t d4 = d >> 2;
  for (int64_t j = tid; j < d4; j += kFwdThreads) {
    float4 xv[kFwdRows];
#pragma unroll
    for (int i = 0; i < kFwdRows; ++i) {
      xv[i] = row0 + i < rows ? __ldg(reinterpret_cast<const float4*>(x + (row0 + i) * d) + j)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      xv[i] = make_float4(relu_if(xv[i].x, x_relu), relu_if(xv[i].y, x_relu), relu_if(xv[i].z, x_relu),
                          relu_if(xv[i].w, x_relu));
    }
#pragma unroll
    for (int o = 0; o < RMAX; ++o) {
      if (o >= r) break;
      const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (int64_t)o * d) + j);
#pragma unroll
      for (int i = 0; i < kFwdRows; ++i) {
        acc[i][o] = fmaf(wv.x, xv[i].x, acc[i][o]);
        acc[i][o] = fmaf(wv.y, xv[i].y, acc[i][o]);
        acc[i][o] = fmaf(wv.z, xv[i].z, acc[i][o]);
        acc[i][o] = fmaf(wv.w, xv[i].w, acc[i][o]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kFwdRows; ++i)
#pragma unroll
    for (int o = 0; o < RMAX; ++o) {
      if (o >= r) break;
      const float v = warp_sum(acc[i][o]);
      if (lane == 0) red[warp][i * RMAX + o] = v;
    }
  __syncthreads();
  for (int e = tid; e < kFwdRows * RMAX; e += kFwdThreads) {
    const int i = e / RMAX, o = e - i * RMAX;
    if (o >= r || row0 + i >= rows) continue;
    float t = red[0][e];
#pragma unroll
    for (int q = 1; q < kFwdThreads / 32; ++q) t += red[q][e];
    y[(row0 + i) * r + o] = (bias ? __ldg(bias + o) : 0.f) + t;
  }
}

struct LinearFwdProb {
  static constexpr bool kAMajorM = false;
  static constexpr bool kBMajorN = false;
  static constexpr bool kExact = false;
  const float* x;
  const float* w;
  const float* bias;
  float* y;
  int x_relu;
  int64_t M, N, K;  // rows, r, d
  __device__ float init(int, int64_t, int64_t n) const { return (bias && n < N) ? __ldg(bias + n) : 0.f; }
  __device__ float a(int, int64_t m, int64_t k) const { return relu_if(__ldg(x + m * K + k), x_relu); }
  __device__ float b(int, int64_t k, int64_t n) const { return __ldg(w + n * K + k); }
  template <int TM, int TN>
  __device__ void epilogue(int, int64_t m0, int64_t n0, int tx, int ty, float (&acc)[TM][TN]) const {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
        if (m < M && n < N) y[m * N + n] = acc[i][j];
      }
  }
};

bool linear_fwd_fuses_dgrad(int64_t d, int64_t r, const float* dx, const float* mask) {
  return (d & 3) == 0 && r <= 16 && (reinterpret_cast<uintptr_t>(dx) & 15) == 0 &&
         (!mask || (reinterpret_cast<uintptr_t>(mask) & 15) == 0);
}

bool linear_fwd_fuses_loss(int64_t d, int64_t r, const float* x, const float* w) {
  return (d & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(w) & 15) == 0 && r <= 64;
}

void launch_linear_fwd(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
                       int64_t rows, int64_t d, int64_t r, float* y, const LossFuse* loss) {
  LossFuse ce{};
  if (loss) {
    if (!linear_fwd_fuses_loss(d, r, x, w)) raise(DPG_ERR_INTERNAL, "linear forward cannot fuse the loss");
    if (loss->dx && !linear_fwd_fuses_dgrad(d, r, loss->dx, loss->dmask))
      raise(DPG_ERR_INTERNAL, "linear forward cannot fuse the input gradient");
    ce = *loss;
    ce.err = ctx->dev_err;
  }
  if (rows == 0) return;
  const bool aligned = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(w) & 15) == 0;
  if (aligned && r <= 64) {
    if (d >= 8192 && r <= 16)
      ::dpg::launch_pdl(linear_fwd_row_kernel<16, 8>, (unsigned)rows, 256, 0, ctx->stream, x, x_relu, w, bias, d, (int)r, y, ce);
    else if (r <= 16) ::dpg::launch_pdl(linear_fwd_row_kernel<16, 4>, (unsigned)rows, 128, 0, ctx->stream, x, x_relu, w, bias, d, (int)r, y, ce);
    else if (r <= 32) ::dpg::launch_pdl(linear_fwd_row_kernel<32, 4>, (unsigned)rows, 128, 0, ctx->stream, x, x_relu, w, bias, d, (int)r, y, ce);
    else ::dpg::launch_pdl(linear_fwd_row_kernel<64, 4>, (unsigned)rows, 128, 0, ctx->stream, x, x_relu, w, bias, d, (int)r, y, ce);
    DPG_LAUNCH_CHECK(ctx);
    return;
  }
  if (aligned && r <= 16) {
    const unsigned g4 = (unsigned)((rows + kFwdRows - 1) / kFwdRows);
    if (r <= 4) ::dpg::launch_pdl(linear_fwd_rows_kernel<4>, g4, kFwdThreads, 0, ctx->stream, x, x_relu, w, bias, rows, d, (int)r, y);
    else ::dpg::launch_pdl(linear_fwd_rows_kernel<16>, g4, kFwdThreads, 0, ctx->stream, x, x_relu, w, bias, rows, d, (int)r, y);
    DPG_LAUNCH_CHECK(ctx);
    return;
  }
  const unsigned grid = (unsigned)((rows + 7) / 8);
  if (r <= 4) {
    ::dpg::launch_pdl(linear_fwd_narrow_kernel<4>, grid, 256, 0, ctx->stream, x, x_relu, w, bias, rows, d, (int)r, y);
  } else if (r <= 16) {
    ::dpg::launch_pdl(linear_fwd_narrow_kernel<16>, grid, 256, 0, ctx->stream, x, x_relu, w, bias, rows, d, (int)r, y);
  } else if (r <= 32) {
    ::dpg::launch_pdl(linear_fwd_narrow_kernel<32>, grid, 256, 0, ctx->stream, x, x_relu, w, bias, rows, d, (int)r, y);
  } else {
    LinearFwdProb p{x, w, bias, y, x_relu, rows, r, d};
    launch_igemm<64, 64, 16>(ctx, p, 1);
    return;
  }
  DPG_LAUNCH_CHECK(ctx);
}

// linear dgrad (layers.hpp:606-625): dx[row, j] = sum_o dy[row, o] W[o, j], o ascending, with
// the ReLU mask of the producing layer.
__global__ void __launch_bounds__(256) linear_dgrad_kernel(const float* __restrict__ dy,
                                                           const float* __restrict__ w,
                                                           int64_t rows, int64_t d, int64_t r,
                                                           const float* __restrict__ mask,
                                                           float* __restrict__ dx) {
  pdl_wait();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * d) return;
  // 32-bit division when the index fits (the common case; int64 division is a long sequence)
  const int64_t row = (rows * d < (int64_t(1) << 31)) ? (int64_t)((uint32_t)e / (uint32_t)d) : e / d;
  const int64_t j = e - row * d;
  float acc = 0.f;
  for (int64_t o = 0; o < r; ++o) acc = fmaf(__ldg(dy + row * r + o), __ldg(w + o * d + j), acc);
  if (mask && !(__ldg(mask + e) > 0.f)) acc = 0.f;
  dx[e] = acc;
}

// d % 4 == 0, r <= RMAX: blockIdx.y = row, each thread 4 consecutive j (128-bit loads of W and the
// mask, one 128-bit store), the row's r highway values in registers
template <int RMAX>
__global__ void __launch_bounds__(256) linear_dgrad_vec_kernel(const float* __restrict__ dy,
                                                               const float* __restrict__ w, int64_t d,
                                                               int r, const float* __restrict__ mask,
                                                               float* __restrict__ dx) {
  pdl_wait();
  const int64_t row = blockIdx.y;
  const int64_t j = 4 * ((int64_t)blockIdx.x * 256 + threadIdx.x);
  if (j >= d) return;
  float dv[RMAX];
#pragma unroll
  for (int o = 0; o < RMAX; ++o) dv[o] = o < r ? __ldg(dy + row * r + o) : 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int o = 0; o < RMAX; ++o) {
    if (o >= r) break;
    const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (int64_t)o * d + j));
    acc.x = fmaf(dv[o], wv.x, acc.x);
    acc.y = fmaf(dv[o], wv.y, acc.y);
    acc.z = fmaf(dv[o], wv.z, acc.z);
    acc.w = fmaf(dv[o], wv.w, acc.w);
  }
  if (mask) {
    const float4 mv = __ldg(reinterpret_cast<const float4*>(mask + row * d + j));
    if (!(mv.x > 0.f)) acc.x = 0.f;
    if (!(mv.y > 0.f)) acc.y = 0.f;
    if (!(mv.z > 0.f)) acc.z = 0.f;
    if (!(mv.w > 0.f)) acc.w = 0.f;
  }
  *reinterpret_cast<float4*>(dx + row * d + j) = acc;
}

void launch_linear_dgrad(dpg_ctx* ctx, const float* dy, const float* w, int64_t rows, int64_t d,
                         int64_t r, const float* mask_src, float* dx) {
  const int64_t n = rows * d;
  if (n == 0) return;
  const bool aligned = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(dx) & 15) == 0 &&
                       (!mask_src || (reinterpret_cast<uintptr_t>(mask_src) & 15) == 0);
  if (aligned && r <= 16 && rows < 65536) {
    const dim3 grid((unsigned)((d / 4 + 255) / 256), (unsigned)rows);
    if (r <= 4)
      ::dpg::launch_pdl(linear_dgrad_vec_kernel<4>, grid, 256, 0, ctx->stream, dy, w, d, (int)r, mask_src, dx);
    else
      ::dpg::launch_pdl(linear_dgrad_vec_kernel<16>, grid, 256, 0, ctx->stream, dy, w, d, (int)r, mask_src, dx);
    DPG_LAUNCH_CHECK(ctx);
    return;
  }
  ::dpg::launch_pdl(linear_dgrad_kernel, (unsigned)((n + 255) / 256), 256, 0, ctx->stream, dy, w, rows, d, r, mask_src, dx);
  DPG_LAUNCH_CHECK(ctx);
}

// embedding forward (layers.hpp:414-431) from the sorted (id, position) lists: one warp per token.
__global__ void __launch_bounds__(256) embedding_fwd_kernel(const int32_t* __restrict__ sorted_v,
                                                            const int32_t* __restrict__ sorted_s,
                                                            const float* __restrict__ table,
                                                            int64_t total, int64_t t, int64_t dim,
                                                            float* __restrict__ out) {
  pdl_wait();
  const int64_t tok = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (tok >= total) return;
  const int64_t n = tok / t;
  const int64_t v = sorted_v[tok], s = sorted_s[tok];
  const float* src = table + v * dim;
  float* dst = out + (n * t + s) * dim;
  if ((dim & 3) == 0) {
    for (int64_t d0 = 4 * lane; d0 < dim; d0 += 128)
      *reinterpret_cast<float4*>(dst + d0) = __ldg(reinterpret_cast<const float4*>(src + d0));
  } else {
    for (int64_t d0 = lane; d0 < dim; d0 += 32) dst[d0] = __ldg(src + d0);
  }
}

void launch_embedding_fwd(dpg_ctx* ctx, const int32_t* sorted_v, const int32_t* sorted_s,
                          const float* table, int64_t b, int64_t t, int64_t dim, float* out) {
  const int64_t total = b * t;
  if (total == 0) return;
  ::dpg::launch_pdl(embedding_fwd_kernel, (unsigned)((total + 7) / 8), 256, 0, ctx->stream, sorted_v, sorted_s, table, total, t, dim, out);
  DPG_LAUNCH_CHECK(ctx);
}

__global__ void __launch_bounds__(256) softmax_ce_kernel(const float* __restrict__ logits, int logits_relu,
                                                         const float* __restrict__ targets, int64_t b,
                                                         int64_t k, float* __restrict__ loss,
                                                         float* __restrict__ grad, DeviceErr* err) {
  pdl_wait();
  const int64_t n = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (n >= b) return;
  softmax_ce_warp(logits + n * k, logits_relu, targets, n, k, loss, grad, err);
}

void launch_softmax_ce(dpg_ctx* ctx, const float* logits, int logits_relu, const float* targets,
                       int64_t b, int64_t k, float* loss, float* grad) {
  if (b == 0) return;
  ::dpg::launch_pdl(softmax_ce_kernel, (unsigned)((b + 7) / 8), 256, 0, ctx->stream, logits, logits_relu, targets, b, k, loss, grad, ctx->dev_err);
  DPG_LAUNCH_CHECK(ctx);
}

__global__ void relu_mask_kernel(float* __restrict__ g, const float* __restrict__ m, int64_t n) {
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !(m[i] > 0.f)) g[i] = 0.f;
}

void launch_relu_mask(dpg_ctx* ctx, float* g, const float* mask_src, int64_t n) {
  if (n == 0) return;
  ::dpg::launch_pdl(relu_mask_kernel, (unsigned)((n + 255) / 256), 256, 0, ctx->stream, g, mask_src, n);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace dpg
