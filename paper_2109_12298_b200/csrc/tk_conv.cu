// tk_conv.cu — "thin-K" conv layers (ic * kh * kw <= 64, e.g. an RGB or greyscale input layer) on CUDA cores.
//
//   per-sample   G[n][oc][k]   = sum_p B[n, oc, p] X~[n, k, p]  + ||G_n||^2     (grad_sample.hpp:135-150)
//                gb[n][oc]     = (float) sum_p (double) B[n, oc, p] + ||gb_n||^2 (sum_middle, tensor.hpp:197-205)
//   clipped sum  S_z[oc][k]    = sum_{n in split z} s_n G_n[oc][k]              (optimizer.hpp:99-114)
//
// With K <= 32 the per-sample gradient is a (oc x K) matrix — a quarter of a UMMA tile's 128 rows
// — summed over P positions: the tensor-core pipeline's per-stage cost (gather + hi/lo split +
// smem stores for 16 K) buys ~1/4 useful rows, so the rule and the clipped sum run as direct
// contractions from shared memory instead (measured, CIFAR conv1 b=512: rule + bias rule
// 28 + 12 -> 31 us, clipped sum 52 -> 34 us); the forward runs on CUDA cores too (layers.cu
// conv_fwd_thin_kernel, compile-time shaped: 30 -> 23 us against the register-gather tcgen05 kernel). One CTA
// stages one sample's zero-padded image (ReLU applied) once; every im2col element is then a
// shared-memory read at (window origin of p) + (tap offset of k), no bounds checks.
//
// The clipped sum is formed per sample from G_n computed in registers (never re-read from HBM),
// scaled by s_n and accumulated over the CTA's samples in the reference's order (ascending n);
// splits are combined in fixed order by splitk_reduce.
#include <algorithm>
#include <cstdlib>

#include "conv_common.cuh"

namespace dpg {
namespace tk {

constexpr int kThreads = 256;
constexpr int kMaxK = 64;
constexpr int kMaxOc = 64;

struct Geo {
  int ic, h, w, oc, kh, kw, stride, pad, oh, ow, P, Kc, hp, wp;
  int hw_nhwc;  // the highway arrives channels-last [b][P][oc] (the engine's TMA-fed dgrad output)
};

Geo make(const ConvGeom& g) {
  Geo r;
  r.ic = (int)g.ic; r.h = (int)g.h; r.w = (int)g.w; r.oc = (int)g.oc;
  r.kh = (int)g.kh; r.kw = (int)g.kw; r.stride = (int)g.stride; r.pad = (int)g.pad;
  r.oh = (int)g.oh; r.ow = (int)g.ow; r.P = (int)g.P(); r.Kc = (int)g.K();
  // padded extent covering every window: (o - 1) * stride + k
  r.hp = std::max<int>(r.h + 2 * r.pad, (r.oh - 1) * r.stride + r.kh);
  r.wp = std::max<int>(r.w + 2 * r.pad, (r.ow - 1) * r.stride + r.kw);
  r.hw_nhwc = 0;
  return r;
}

// Shared-memory plan (floats / ints): padded image, tap table, position table.
struct Plan {
  int xs, kt, pb;
};
__host__ __device__ inline Plan plan(const Geo& g) {
  Plan p;
  p.xs = (g.ic * g.hp * g.wp + 3) & ~3;
  p.kt = kMaxK;
  p.pb = (g.P + 3) & ~3;
  return p;
}

// stage sample n's image zero-padded (ReLU of the stored pre-activation when relu) + tables.
// The interior is copied with every thread's loads issued before any store (8 in flight per
// thread per round): a load-use chain per element would serialise HBM latencies.
__device__ __forceinline__ void stage_image(const Geo& g, const float* __restrict__ x, int relu, int64_t n,
                                            float* xs, int* kt, int* pb) {
  const int tid = threadIdx.x;
  const int hw = g.h * g.w, tot = g.ic * hw;
  if (g.hp != g.h || g.wp != g.w)
    for (int i = tid; i < g.ic * g.hp * g.wp; i += kThreads) xs[i] = 0.f;
  __syncthreads();
  // one warp per image row (c, yy), lanes along xx; four rows' loads in flight per lane
  const float* xn = x + n * (int64_t)tot;
  const int lane = tid & 31, warp = tid >> 5, nrows = g.ic * g.h;
  for (int r0 = warp; r0 < nrows; r0 += 4 * (kThreads / 32)) {
    for (int x0 = 0; x0 < g.w; x0 += 32) {
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + j * (kThreads / 32), xx = x0 + lane;
        v[j] = (r < nrows && xx < g.w) ? __ldg(xn + (int64_t)r * g.w + xx) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + j * (kThreads / 32), xx = x0 + lane;
        if (r < nrows && xx < g.w) {
          const int c = r / g.h, yy = r - c * g.h;
          xs[(c * g.hp + yy + g.pad) * g.wp + xx + g.pad] = relu_if(v[j], relu);
        }
      }
    }
  }
  if (tid < kMaxK) {
    int off = 0;
    if (tid < g.Kc) {
      const int khw = g.kh * g.kw;
      const int c = tid / khw, r = tid - c * khw;
      const int ki = r / g.kw, kj = r - ki * g.kw;
      off = (c * g.hp + ki) * g.wp + kj;
    }
    kt[tid] = off;  // k >= Kc: a valid address whose products are dropped
  }
  for (int p = tid; p < g.P; p += kThreads) {
    const int oy = p / g.ow, ox = p - oy * g.ow;
    pb[p] = oy * g.stride * g.wp + ox * g.stride;
  }
}

// ------------------------------------------------------------------------------ per-sample G
// Work split: tiles of 4 oc x 4 k (og, kg) times `parts` slices of the positions; thread t owns
// tile t % tiles, slice t / tiles, and 16 accumulators. The highway rows are staged transposed
// ([p][oc], 128-bit broadcast reads); slices are combined in fixed order through shared memory.
// (Measured against a variant that materialises the im2col as Xc[p][k] with 4 x 8 tiles: fewer
// instructions but one more staging phase and 3 instead of 4 CTAs per SM, 31 -> 43 us.)
struct GsPlan {
  int tiles, parts, kg, ocp;
};
__host__ __device__ inline GsPlan gs_plan(const Geo& g) {
  GsPlan q;
  q.kg = (g.Kc + 3) / 4;
  q.tiles = (g.oc / 4) * q.kg;
  q.parts = kThreads / q.tiles;
  if (q.parts > 8) q.parts = 8;
  q.ocp = g.oc + 4;  // row stride of the transposed highway tile (bank spread)
  return q;
}

// G_n into gsm[oc][Kc] (shared); also the bias record of sample n when gb (GS mode) and its
// squared norm in bsq (lane 0 of each warp: its rows' share). Caller syncs before reading gsm.
__device__ __forceinline__ void sample_g(const Geo& g, const GsPlan& q, const float* __restrict__ x, int relu,
                                         const float* __restrict__ hw, int64_t n, float* xs, int* kt,
                                         int* pb, float* bs, float* gsm, float* gb, bool bias_norm,
                                         double& bsq) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  stage_image(g, x, relu, n, xs, kt, pb);
  const float* hn = hw + n * (int64_t)g.oc * g.P;
  if (g.hw_nhwc) {
    // channels-last highway: already the [p][oc] order of the tile (oc % 4 == 0): 16-byte copies,
    // 4 in flight per thread
    const int oc4 = g.oc / 4, tot4 = g.P * oc4;
    const float4* h4 = reinterpret_cast<const float4*>(hn);
    for (int i0 = tid; i0 < tot4; i0 += 4 * kThreads) {
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + j * kThreads;
        v[j] = i < tot4 ? __ldg(h4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + j * kThreads;
        if (i < tot4) {
          const int m = i / oc4, c4 = i - m * oc4;
          *reinterpret_cast<float4*>(bs + m * q.ocp + 4 * c4) = v[j];
        }
      }
    }
  }
  // one warp per highway row, lanes along p, 8 loads in flight per lane; transposed stores
  for (int o = warp; o < g.oc && !g.hw_nhwc; o += kThreads / 32) {
    const float* row = hn + (int64_t)o * g.P;
    for (int m0 = 0; m0 < g.P; m0 += 8 * 32) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int m = m0 + 32 * j + lane;
        v[j] = m < g.P ? __ldg(row + m) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int m = m0 + 32 * j + lane;
        if (m < g.P) bs[m * q.ocp + o] = v[j];
      }
    }
  }
  __syncthreads();
  // bias rule: each row summed in fp64 with gs_bias_kernel's association (lane-strided, then a
  // fixed shuffle tree), so its records are bit-identical to the generic bias kernel's
  bsq = 0.0;
  if (gb || bias_norm) {
    for (int o = warp; o < g.oc; o += kThreads / 32) {
      double acc = 0.0;
      for (int m = lane; m < g.P; m += 32) acc += (double)bs[m * q.ocp + o];
      acc = warp_sum(acc);
      const float v = (float)acc;
      if (lane == 0) {
        if (gb) gb[n * g.oc + o] = v;
        bsq += (double)v * v;
      }
    }
  }
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const int tile = tid % q.tiles, part = tid / q.tiles;
  const int og = tile / q.kg, kg = tile - og * q.kg;
  if (part < q.parts) {
    const int per = ((g.P + q.parts - 1) / q.parts + 3) & ~3;  // slices start at multiples of 4
    const int p0 = min(g.P, part * per), p1 = min(g.P, p0 + per);
    const int k0 = 4 * kg;
    const int o1 = kt[k0], o2 = kt[min(k0 + 1, kMaxK - 1)], o3 = kt[min(k0 + 2, kMaxK - 1)],
              o4 = kt[min(k0 + 3, kMaxK - 1)];
    auto step = [&](int pbase, const float4& b) {
      const float* xp = xs + pbase;
      const float xv[4] = {xp[o1], xp[o2], xp[o3], xp[o4]};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[0][j] = fmaf(b.x, xv[j], acc[0][j]);
        acc[1][j] = fmaf(b.y, xv[j], acc[1][j]);
        acc[2][j] = fmaf(b.z, xv[j], acc[2][j]);
        acc[3][j] = fmaf(b.w, xv[j], acc[3][j]);
      }
    };
    int p = p0;
    for (; p + 4 <= p1; p += 4) {
      const int4 pb4 = *reinterpret_cast<const int4*>(pb + p);
      step(pb4.x, *reinterpret_cast<const float4*>(bs + (p + 0) * q.ocp + 4 * og));
      step(pb4.y, *reinterpret_cast<const float4*>(bs + (p + 1) * q.ocp + 4 * og));
      step(pb4.z, *reinterpret_cast<const float4*>(bs + (p + 2) * q.ocp + 4 * og));
      step(pb4.w, *reinterpret_cast<const float4*>(bs + (p + 3) * q.ocp + 4 * og));
    }
    for (; p < p1; ++p) step(pb[p], *reinterpret_cast<const float4*>(bs + p * q.ocp + 4 * og));
  }
  __syncthreads();  // bs is reused as the slice buffer
  float* red = bs;  // [parts][oc][Kc]
  const int ne = g.oc * g.Kc;
  if (part < q.parts) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * kg + j < g.Kc) red[part * ne + (4 * og + i) * g.Kc + 4 * kg + j] = acc[i][j];
  }
  __syncthreads();
  for (int e = tid; e < ne; e += kThreads) {
    float v = red[e];
    for (int s = 1; s < q.parts; ++s) v += red[s * ne + e];
    gsm[e] = v;
  }
}

size_t gs_smem(const Geo& g) {
  const Plan pl = plan(g);
  const GsPlan q = gs_plan(g);
  const size_t bs = std::max<size_t>((size_t)g.P * q.ocp, (size_t)q.parts * g.oc * g.Kc);
  return sizeof(float) * ((size_t)pl.xs + pl.kt + pl.pb + ((bs + 3) & ~size_t(3)) + (size_t)g.oc * g.Kc) + 64;
}

// MODE 0: G record + norm partial + bias rule (one sample per CTA)
// MODE 1: clipped-sum partial of split z (samples [z spl, (z + 1) spl))
template <int MODE>
__global__ void __launch_bounds__(kThreads) tk_gs_kernel(Geo g, const float* __restrict__ x, int relu,
                                                         const float* __restrict__ hw,
                                                         const float* __restrict__ scale, int64_t b,
                                                         int64_t spl, float* __restrict__ out,
                                                         double* __restrict__ sq_part, float* __restrict__ gb,
                                                         double* __restrict__ sq_b) {
  pdl_wait();
  extern __shared__ __align__(16) float sm[];
  __shared__ double red[kThreads / 32];
  __shared__ double bred[kThreads / 32];
  const Plan pl = plan(g);
  const GsPlan q = gs_plan(g);
  float* xs = sm;
  int* kt = reinterpret_cast<int*>(xs + pl.xs);
  int* pb = kt + pl.kt;
  float* bs = reinterpret_cast<float*>(pb + pl.pb);
  const int bsz = std::max(g.P * q.ocp, q.parts * g.oc * g.Kc);
  float* gsm = bs + ((bsz + 3) & ~3);
  const int ne = g.oc * g.Kc, tid = threadIdx.x;
  if (MODE == 0) {
    const int64_t n = blockIdx.x;
    double bsq;
    sample_g(g, q, x, relu, hw, n, xs, kt, pb, bs, gsm, gb, sq_b != nullptr, bsq);
    __syncthreads();
    double sq = 0.0;
    float* gn = out ? out + n * (int64_t)ne : nullptr;
    for (int e = tid; e < ne; e += kThreads) {
      const float v = gsm[e];
      if (gn) st_stream(gn + e, v);
      sq += (double)v * v;
    }
    const double t = block_sum<kThreads>(sq, red);
    // the bias norm with gs_bias_kernel's reduction (lane 0 of each warp holds its rows' sum)
    const double tb = block_sum<kThreads>(bsq, bred);
    if (tid == 0) {
      if (sq_part) sq_part[n] = t;
      if (sq_b) sq_b[n] = tb;
    }
  } else {
    const int64_t z = blockIdx.x;
    constexpr int kPer = (kMaxK * kMaxOc + kThreads - 1) / kThreads;
    float acc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] = 0.f;
    const int64_t n_end = std::min<int64_t>(b, (z + 1) * spl);
    for (int64_t n = z * spl; n < n_end; ++n) {
      double bsq;
      sample_g(g, q, x, relu, hw, n, xs, kt, pb, bs, gsm, nullptr, false, bsq);
      __syncthreads();
      const float s = __ldg(scale + n);
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int e = tid + j * kThreads;
        if (e < ne) acc[j] = fmaf(s, gsm[e], acc[j]);
      }
      __syncthreads();  // every buffer is reused by the next sample
    }
    float* part = out + z * (int64_t)ne;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int e = tid + j * kThreads;
      if (e < ne) part[e] = acc[j];
    }
  }
}

bool supported(const ConvGeom& cg) {
  if (cg.K() > kMaxK || cg.oc > kMaxOc || cg.oc % 4 != 0 || cg.P() <= 0) return false;
  return gs_smem(make(cg)) <= 160 * 1024;
}

static void set_smem(const void* fn, size_t bytes) { ensure_smem_attr(fn, (int)bytes); }

void gs(dpg_ctx* ctx, const float* x, int relu, const float* hw, const ConvGeom& cg, float* gw,
        double* sq_part, float* gb, double* sq_b, bool hw_nhwc) {
  Geo g = make(cg);
  g.hw_nhwc = hw_nhwc ? 1 : 0;
  const size_t smem = gs_smem(g);
  set_smem((const void*)tk_gs_kernel<0>, smem);
  ::dpg::launch_pdl(tk_gs_kernel<0>, (unsigned)cg.b, kThreads, smem, ctx->stream, g, x, relu, hw, nullptr, cg.b, 1, gw,
                                                                    sq_part, gb, sq_b);
  DPG_LAUNCH_CHECK(ctx);
}

int csum_splits(const ConvGeom& cg) {
  const int64_t want = std::min<int64_t>(cg.b, 4 * kNumSMs);
  const int64_t spl = (cg.b + want - 1) / std::max<int64_t>(1, want);
  return (int)((cg.b + spl - 1) / std::max<int64_t>(1, spl));
}

void csum(dpg_ctx* ctx, const float* x, int relu, const float* hw, const float* scale, const ConvGeom& cg,
          float* part, int splits, bool hw_nhwc) {
  Geo g = make(cg);
  g.hw_nhwc = hw_nhwc ? 1 : 0;
  const size_t smem = gs_smem(g);
  const int64_t spl = (cg.b + splits - 1) / splits;
  set_smem((const void*)tk_gs_kernel<1>, smem);
  ::dpg::launch_pdl(tk_gs_kernel<1>, (unsigned)splits, kThreads, smem, ctx->stream, g, x, relu, hw, scale, cg.b, spl, part,
                                                                      nullptr, nullptr, nullptr);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace tk
}  // namespace dpg
