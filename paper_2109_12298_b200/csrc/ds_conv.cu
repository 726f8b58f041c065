// ds_conv.cu — direct per-sample conv contractions (no shared memory, no block barriers).
//
//   GS   : G[n][oc][kcol] = sum_p B[n, oc, p] X~[n, kcol, p]    (per_sample_rule_conv2d,
//          grad_sample.hpp:135-150) with the fused ||G_n||^2 partial
//   CSUM : S[oc][kcol]    = sum_n s_n sum_p B[n, oc, p] X~[n, kcol, p]   (clip_and_sum pass 2,
//          optimizer.hpp:99-114) accumulated without materialising G
//
// Each thread owns a 4 (oc) x 4 (kcol) block of one sample's G: it reads its four highway rows
// with 128-bit loads, gathers its four im2col columns straight from x (L1-resident: one sample's
// image is a few KB), keeps 16 accumulators, and writes four 128-bit streaming stores — the
// per-sample gradient is the largest HBM stream of the step and is written exactly once.
// Consecutive threads own consecutive kcol quads, so every warp store covers 512 contiguous
// bytes. No shared memory and no barriers (except the final norm reduction) keeps occupancy
// high enough to cover load latency with many independent warps.
//
// With kExact the p-sum is the reference's sequential `acc = acc + b * x` (two roundings,
// tensor.hpp:324-336), reproducing its per-sample gradient bits; used where the layer is store-
// bound anyway (small P).
#include <cstdlib>

#include "conv_common.cuh"

namespace dpg {
namespace ds {

constexpr int kThreads = 256;

struct Params {
  const float* x;
  int relu;
  const float* hw;
  const float* scale;  // CSUM
  float* out;          // GS: G [b, oc, Kc]; CSUM: partials [splits, oc, Kc]
  double* sq_part;     // GS: [gridDim.x, b]
  int64_t b, spl;
  int ic, h, w, oc, kh, kw, stride, pad, oh, ow, P, Kc, nq, ng;
};

template <int MODE, bool EXACT>
__global__ void __launch_bounds__(kThreads) ds_conv_kernel(const Params p) {
  pdl_wait();
  const int blk = blockIdx.x * kThreads + threadIdx.x;
  const bool active = blk < p.nq * p.ng;
  const int jq = active ? blk % p.nq : 0, gq = active ? blk / p.nq : 0;
  const int k0 = 4 * jq, oc0 = 4 * gq;
  const int hwsz = p.h * p.w;
  // im2col column offsets of the thread's four kcols: c*h*w + (ki - pad)*w + (kj - pad)
  int koff[4], kiy[4], kix[4];
  bool kval[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = k0 + j;
    kval[j] = active && k < p.Kc;
    const int kk = kval[j] ? k : 0;
    const int khw = p.kh * p.kw;
    const int c = kk / khw, r = kk - c * khw;
    const int ki = r / p.kw, kj = r - ki * p.kw;
    kiy[j] = ki - p.pad;
    kix[j] = kj - p.pad;
    koff[j] = c * hwsz + kiy[j] * p.w + kix[j];
  }
  bool oval[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) oval[i] = active && oc0 + i < p.oc;
  const bool vec4 = (p.P & 3) == 0;

  const int n_begin = (int)(MODE == 0 ? blockIdx.y : blockIdx.y * p.spl);
  const int n_end = (int)(MODE == 0 ? blockIdx.y + 1 : min((int64_t)(blockIdx.y + 1) * p.spl, p.b));
  float tot[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) tot[i][j] = 0.f;
  double sq = 0.0;

  for (int n = n_begin; n < n_end && active; ++n) {
    const float* xn = p.x + (int64_t)n * p.ic * hwsz;
    const float* hn = p.hw + ((int64_t)n * p.oc + oc0) * p.P;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    int oy = 0, ox = 0;
    for (int p0 = 0; p0 < p.P; p0 += 4) {
      float hv[4][4];  // [oc][p]
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (vec4) {
          const float4 v = oval[i] ? __ldg(reinterpret_cast<const float4*>(hn + (int64_t)i * p.P + p0))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          hv[i][0] = v.x; hv[i][1] = v.y; hv[i][2] = v.z; hv[i][3] = v.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            hv[i][e] = (oval[i] && p0 + e < p.P) ? __ldg(hn + (int64_t)i * p.P + p0 + e) : 0.f;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (p0 + e < p.P) {
          const int by = oy * p.stride, bx = ox * p.stride;
          float xv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int iy = by + kiy[j], ix = bx + kix[j];
            xv[j] = (kval[j] && (unsigned)iy < (unsigned)p.h && (unsigned)ix < (unsigned)p.w)
                        ? relu_if(__ldg(xn + koff[j] + by * p.w + bx), p.relu)
                        : 0.f;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (EXACT) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(hv[i][e], xv[j]));
              else acc[i][j] = fmaf(hv[i][e], xv[j], acc[i][j]);
            }
          if (++ox == p.ow) {
            ox = 0;
            ++oy;
          }
        }
      }
    }
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (!oval[i]) continue;
        float* row = p.out ? p.out + ((int64_t)n * p.oc + oc0 + i) * p.Kc + k0 : nullptr;
        if (row && (p.Kc & 3) == 0) {
          st_stream4(row, make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]));
        } else if (row) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (kval[j]) st_stream(row + j, acc[i][j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (kval[j]) sq += (double)acc[i][j] * acc[i][j];
      }
    } else {
      const float sn = __ldg(p.scale + n);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) tot[i][j] = fmaf(sn, acc[i][j], tot[i][j]);
    }
  }
  if (MODE == 0) {
    __shared__ double red[kThreads / 32];
    const double t = block_sum<kThreads>(sq, red);
    if (threadIdx.x == 0 && p.sq_part) p.sq_part[(int64_t)blockIdx.x * p.b + blockIdx.y] = t;
  } else if (active) {
    float* base = p.out + (int64_t)blockIdx.y * p.oc * p.Kc;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!oval[i]) continue;
      float* row = base + (int64_t)(oc0 + i) * p.Kc + k0;
      if ((p.Kc & 3) == 0) {
        *reinterpret_cast<float4*>(row) = make_float4(tot[i][0], tot[i][1], tot[i][2], tot[i][3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (kval[j]) row[j] = tot[i][j];
      }
    }
  }
}

inline Params make_params(const float* x, int relu, const float* hw, const ConvGeom& g) {
  Params p{};
  p.x = x; p.relu = relu; p.hw = hw;
  p.b = g.b;
  p.ic = (int)g.ic; p.h = (int)g.h; p.w = (int)g.w; p.oc = (int)g.oc;
  p.kh = (int)g.kh; p.kw = (int)g.kw; p.stride = (int)g.stride; p.pad = (int)g.pad;
  p.oh = (int)g.oh; p.ow = (int)g.ow; p.P = (int)g.P(); p.Kc = (int)g.K();
  p.nq = (p.Kc + 3) / 4;
  p.ng = (p.oc + 3) / 4;
  return p;
}

bool enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DPG_DS");
    return e && e[0] == '1';
  }();
  return on;
}

int gs_rows(const ConvGeom& g) {
  const Params p = make_params(nullptr, 0, nullptr, g);
  return (p.nq * p.ng + kThreads - 1) / kThreads;
}

void gs(dpg_ctx* ctx, const float* x, int relu, const float* hw, const ConvGeom& g, float* gw,
        double* sq_part) {
  Params p = make_params(x, relu, hw, g);
  p.out = gw;
  p.sq_part = sq_part;
  dim3 grid((unsigned)gs_rows(g), (unsigned)g.b);
  if (p.P <= 16) ::dpg::launch_pdl(ds_conv_kernel<0, true>, grid, kThreads, 0, ctx->stream, p);
  else ::dpg::launch_pdl(ds_conv_kernel<0, false>, grid, kThreads, 0, ctx->stream, p);
  DPG_LAUNCH_CHECK(ctx);
}

int csum_splits(const ConvGeom& g) {
  const Params p = make_params(nullptr, 0, nullptr, g);
  const int64_t threads = (int64_t)p.nq * p.ng;
  // aim for ~32 resident warps per SM worth of threads
  int64_t splits = (int64_t)kNumSMs * 1024 / std::max<int64_t>(1, threads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(splits, g.b));
}

void csum(dpg_ctx* ctx, const float* x, int relu, const float* hw, const float* scale,
          const ConvGeom& g, float* part, int splits) {
  Params p = make_params(x, relu, hw, g);
  p.scale = scale;
  p.out = part;
  p.spl = (g.b + splits - 1) / splits;
  dim3 grid((unsigned)((p.nq * p.ng + kThreads - 1) / kThreads), (unsigned)splits);
  ::dpg::launch_pdl(ds_conv_kernel<1, false>, grid, kThreads, 0, ctx->stream, p);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace ds
}  // namespace dpg
