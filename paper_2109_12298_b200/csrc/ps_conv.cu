// ps_conv.cu — per-sample conv contractions with the sample staged in shared memory.
//
//   GS   : G[n][oc][kcol] = sum_p B[n, oc, p] X~[n, kcol, p]   (per_sample_rule_conv2d,
//          grad_sample.hpp:135-150) + the fused ||G_n||^2 partial, and (optionally) the bias rule
//          gb[n][oc] = sum_p B[n, oc, p] (grad_sample.hpp:146-148, sum_middle order) with its norm
//   CSUM : S[oc][kcol]    = sum_n s_n sum_p B[n, oc, p] X~[n, kcol, p]   (clip_and_sum pass 2,
//          optimizer.hpp:99-114, without materialising G)
//
// One CTA owns an oc tile (`oct` channels) and one sample (GS) or a contiguous group of samples
// (CSUM). Every thread owns exactly ONE register block — 8 output channels x 4 consecutive kcol
// (32 accumulators) — and, when a sample has many positions and few outputs (conv1: 864 outputs,
// 256 positions), one of S position slices of it, reduced through shared memory in slice order.
// One block per thread keeps register use low, so several CTAs stay resident per SM and their
// staging, compute and store phases overlap.
//
// Per sample: the highway rows of the oc tile are staged transposed ([p][oct], so eight channels
// are two 128-bit reads), im2col is expanded one chunk of positions at a time into [p][Kc4]
// (four consecutive kcol = one 128-bit read), gathered from x_n through L1. GS writes each block
// with 128-bit streaming stores — the per-sample gradient is the dominant HBM stream of the step,
// written exactly once — and accumulates its squares in fp64.
//
// These shapes (P = positions per sample <= 256, a few thousand outputs per sample) are
// store- or latency-bound, not tensor-bound.
#include <algorithm>
#include <cstdlib>

#include "conv_common.cuh"

namespace dpg {
namespace ps {

constexpr int kMaxThreads = 320;
constexpr int kTargetItems = 320;           // register blocks per CTA (= threads when S == 1)
constexpr int kChunkBytes = 40 * 1024;      // im2col chunk budget

struct Params {
  const float* x;
  int relu;
  const float* hw;
  const float* scale;  // CSUM
  float* out;          // GS: G [b, oc, Kc]; CSUM: partials [splits, oc, Kc]
  double* sq_part;     // GS: [tiles, b]
  float* gb;           // GS: bias record [b, oc] (nullptr: no bias rule)
  double* sq_b;        // GS: bias norm partials [tiles, b]
  int with_bias;       // GS: bias rule on
  int64_t b, spl;
  int ic, h, w, oc, kh, kw, stride, pad, oh, ow, P, Kc, Kc4;
  int oct, nitems, S, pc, nth;
};

__device__ __forceinline__ double block_sum_dyn(double v, double* red /* >= 32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

template <int MODE>
__global__ void __launch_bounds__(kMaxThreads, 3) ps_conv_kernel(const Params p) {
  pdl_wait();
  extern __shared__ __align__(16) float sm[];
  float* hs = sm;                                             // [P][oct]
  float* xt = hs + p.P * p.oct;                               // [pc][Kc4]
  int* kt = reinterpret_cast<int*>(xt + p.pc * p.Kc4);        // [Kc4] packed (c, ki, kj)
  int* pt = kt + p.Kc4;                                       // [P] packed (by, bx)
  float* red = reinterpret_cast<float*>(pt + ((p.P + 3) & ~3));  // [S-1][32][nitems]
  __shared__ double dred[32];

  const int tid = threadIdx.x, nth = blockDim.x;
  const int item = tid % p.nitems, s = tid / p.nitems;
  const bool active = s < p.S;
  const int nq = p.Kc4 >> 2;
  const int q4 = item % nq, g = item / nq;
  const int oc0 = blockIdx.x * p.oct;
  const int hwsz = p.h * p.w;
  const int n_begin = (int)(MODE == 0 ? blockIdx.y : blockIdx.y * p.spl);
  const int n_end = (int)(MODE == 0 ? blockIdx.y + 1 : min((int64_t)(blockIdx.y + 1) * p.spl, p.b));

  for (int k = tid; k < p.Kc4; k += nth) {
    int e = -1;
    if (k < p.Kc) {
      const int khw = p.kh * p.kw;
      const int c = k / khw, r = k - c * khw;
      const int ki = r / p.kw, kj = r - ki * p.kw;
      e = (c << 10) | (ki << 5) | kj;  // ic < 2^21, kh, kw < 32
    }
    kt[k] = e;
  }
  for (int q = tid; q < p.P; q += nth) {
    const int oy = q / p.ow, ox = q - oy * p.ow;
    const int by = oy * p.stride - p.pad, bx = ox * p.stride - p.pad;
    pt[q] = (by << 16) | (bx & 0xffff);
  }
  // im2col build mapping: thread -> (kcol, position group)
  const int G = nth >= p.Kc4 ? nth / p.Kc4 : 1;
  const int bk0 = nth >= p.Kc4 ? (tid < G * p.Kc4 ? tid % p.Kc4 : p.Kc4) : tid;
  const int bkstep = nth >= p.Kc4 ? p.Kc4 : nth;
  const int bgrp = nth >= p.Kc4 ? tid / p.Kc4 : 0;

  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  double sq = 0.0, sqb = 0.0;

  for (int n = n_begin; n < n_end; ++n) {
    __syncthreads();  // previous sample fully consumed (and kt/pt ready)
    const float sn = MODE == 1 ? __ldg(p.scale + n) : 1.f;
    for (int i = tid; i < p.oct * p.P; i += nth) {
      const int q = i / p.oct, o = i - q * p.oct;  // conflict-free transposed store; rows hit L1
      float v = 0.f;
      if (oc0 + o < p.oc) v = __ldg(p.hw + ((int64_t)n * p.oc + oc0 + o) * p.P + q);
      hs[q * p.oct + o] = MODE == 1 ? sn * v : v;
    }
    if (MODE == 0 && p.with_bias && tid < p.oct && oc0 + tid < p.oc) {
      // bias rule: (float) sequential fp64 sum over positions (sum_middle, tensor.hpp:197-205)
      double a = 0.0;
      const float* row = p.hw + ((int64_t)n * p.oc + oc0 + tid) * p.P;
#pragma unroll 8
      for (int q = 0; q < p.P; ++q) a += (double)__ldg(row + q);
      const float v = (float)a;
      if (p.gb) p.gb[(int64_t)n * p.oc + oc0 + tid] = v;
      sqb += (double)v * v;
    }
    const float* xn = p.x + (int64_t)n * p.ic * hwsz;
    for (int c0 = 0; c0 < p.P; c0 += p.pc) {
      const int cn = min(p.pc, p.P - c0);
      __syncthreads();  // staging done / previous chunk consumed
      for (int k = bk0; k < p.Kc4; k += bkstep) {
        const int e = kt[k];
        const int coff = (e >> 10) * hwsz, ki = (e >> 5) & 31, kj = e & 31;
        for (int pp = bgrp; pp < cn; pp += G) {
          float v = 0.f;
          if (e >= 0) {
            const int t = pt[c0 + pp];
            const int iy = (t >> 16) + ki, ix = (int)(short)(t & 0xffff) + kj;
            if ((unsigned)iy < (unsigned)p.h && (unsigned)ix < (unsigned)p.w)
              v = relu_if(__ldg(xn + coff + iy * p.w + ix), p.relu);
          }
          xt[pp * p.Kc4 + k] = v;
        }
      }
      __syncthreads();
      if (active) {
        const int lo = p.S > 1 ? s * cn / p.S : 0;
        const int hi = p.S > 1 ? (s + 1) * cn / p.S : cn;
        const float* xr = xt + 4 * q4;
        const float* hr = hs + c0 * p.oct + 8 * g;
#pragma unroll 4
        for (int pp = lo; pp < hi; ++pp) {
          const float4 xv = *reinterpret_cast<const float4*>(xr + pp * p.Kc4);
          const float4 h0 = *reinterpret_cast<const float4*>(hr + pp * p.oct);
          const float4 h1 = *reinterpret_cast<const float4*>(hr + pp * p.oct + 4);
          const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            acc[i][0] = fmaf(hv[i], xv.x, acc[i][0]);
            acc[i][1] = fmaf(hv[i], xv.y, acc[i][1]);
            acc[i][2] = fmaf(hv[i], xv.z, acc[i][2]);
            acc[i][3] = fmaf(hv[i], xv.w, acc[i][3]);
          }
        }
      }
    }
    if (MODE == 0) {
      if (p.S > 1) {
        if (active && s > 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) red[((s - 1) * 32 + i * 4 + j) * p.nitems + item] = acc[i][j];
        }
        __syncthreads();
        if (s == 0) {
          for (int z = 0; z < p.S - 1; ++z)
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) acc[i][j] += red[(z * 32 + i * 4 + j) * p.nitems + item];
        }
      }
      if (s == 0) {
        const int k0 = 4 * q4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int oc = oc0 + 8 * g + i;
          if (oc < p.oc) {
            float* row = p.out ? p.out + ((int64_t)n * p.oc + oc) * p.Kc : nullptr;
            if (row && (p.Kc & 3) == 0) {
              st_stream4(row + k0, make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]));
            } else if (row) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (k0 + j < p.Kc) st_stream(row + k0 + j, acc[i][j]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (k0 + j < p.Kc) sq += (double)acc[i][j] * acc[i][j];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    }
  }
  if (MODE == 1) {
    if (p.S > 1) {
      __syncthreads();
      if (active && s > 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) red[((s - 1) * 32 + i * 4 + j) * p.nitems + item] = acc[i][j];
      }
      __syncthreads();
      if (s == 0) {
        for (int z = 0; z < p.S - 1; ++z)
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] += red[(z * 32 + i * 4 + j) * p.nitems + item];
      }
    }
    float* base = p.out + (int64_t)blockIdx.y * p.oc * p.Kc;
    if (s == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int oc = oc0 + 8 * g + i;
        if (oc < p.oc) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (4 * q4 + j < p.Kc) base[(int64_t)oc * p.Kc + 4 * q4 + j] = acc[i][j];
        }
      }
    }
  } else {
    const double t = block_sum_dyn(sq, dred);
    if (tid == 0 && p.sq_part) p.sq_part[(int64_t)blockIdx.x * p.b + blockIdx.y] = t;
    if (p.with_bias) {
      const double tb = block_sum_dyn(sqb, dred);
      if (tid == 0 && p.sq_b) p.sq_b[(int64_t)blockIdx.x * p.b + blockIdx.y] = tb;
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
  p.Kc4 = (p.Kc + 3) & ~3;
  // oc tile: the largest multiple of 8 whose block count stays near kTargetItems
  const int nq = p.Kc4 / 4;
  const int oc8 = (p.oc + 7) & ~7;
  int oct = 8;
  for (int c : {64, 32, 16}) {
    if (c <= std::max(8, oc8) && nq * (c / 8) <= kTargetItems) {
      oct = std::min(c, oc8);
      break;
    }
  }
  p.oct = oct;
  p.nitems = nq * (oct / 8);
  // position slices when there are few blocks and many positions (reduced in slice order)
  int S = 1;
  while (p.nitems * S * 2 <= 256 && p.P % (2 * S) == 0 && p.P / (2 * S) >= 8) S *= 2;
  p.S = S;
  p.nth = std::min(kMaxThreads, ((p.nitems * S + 31) / 32) * 32);
  if (S > 1) {
    p.pc = p.P;
  } else {
    p.pc = std::max(1, std::min(p.P, kChunkBytes / (4 * p.Kc4)));
  }
  return p;
}

inline size_t smem_bytes(const Params& p) {
  return sizeof(float) * ((size_t)p.P * p.oct + (size_t)p.pc * p.Kc4) +
         sizeof(int) * ((size_t)p.Kc4 + ((p.P + 3) & ~3)) +
         sizeof(float) * (size_t)(p.S - 1) * 32 * p.nitems;
}

// shape check: shared memory fits, index packing, one register block per thread
bool fits(const ConvGeom& g) {
  if (g.kh >= 32 || g.kw >= 32 || g.ic >= (1 << 21)) return false;
  const Params p = make_params(nullptr, 0, nullptr, g);
  if (p.nitems * p.S > kMaxThreads) return false;
  if (g.oh * g.stride + g.kh > 32000 || g.ow * g.stride + g.kw > 32000) return false;
  return smem_bytes(p) <= 160 * 1024;
}

// DPG_PS=0 / DPG_PS=1 force the staged CUDA-core kernels off / on for A/B measurements.
static int force_mode() {
  static const int force = [] {
    const char* e = std::getenv("DPG_PS");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return force;
}

// A/B alternative to rows_conv (P <= 16) and tcgen05 (larger P): forced with DPG_PS=1.
bool supported(const ConvGeom& g) { return force_mode() == 1 && fits(g); }
// the clipped sums stay on tcgen05 unless forced (measured faster there)
bool supported_csum(const ConvGeom& g) { return force_mode() == 1 && fits(g); }

template <int MODE>
static void launch(dpg_ctx* ctx, const Params& p, unsigned gy) {
  const size_t smem = smem_bytes(p);
  dim3 grid((unsigned)((p.oc + p.oct - 1) / p.oct), gy);
  static int attr = 0;
  if ((int)smem > attr) {
    DPG_CUDA(cudaFuncSetAttribute(ps_conv_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  160 * 1024));
    attr = 160 * 1024;
  }
  ::dpg::launch_pdl(ps_conv_kernel<MODE>, grid, p.nth, smem, ctx->stream, p);
  DPG_LAUNCH_CHECK(ctx);
}

int gs_rows(const ConvGeom& g) {
  const Params p = make_params(nullptr, 0, nullptr, g);
  return (int)((g.oc + p.oct - 1) / p.oct);
}

void gs(dpg_ctx* ctx, const float* x, int relu, const float* hw, const ConvGeom& g, float* gw,
        double* sq_part, float* gb, double* sq_b) {
  Params p = make_params(x, relu, hw, g);
  p.out = gw;
  p.sq_part = sq_part;
  p.gb = gb;
  p.sq_b = sq_b;
  p.with_bias = (gb || sq_b) ? 1 : 0;
  launch<0>(ctx, p, (unsigned)g.b);
}

int csum_splits(const ConvGeom& g) {
  const Params p = make_params(nullptr, 0, nullptr, g);
  const int64_t tiles = (g.oc + p.oct - 1) / p.oct;
  // ~4 CTAs per SM (the fixed-order split reduce is cheap next to an idle SM)
  int64_t splits = (4 * kNumSMs + tiles - 1) / tiles;
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, g.b));
  const int64_t spl = (g.b + splits - 1) / splits;
  return (int)std::max<int64_t>(1, (g.b + spl - 1) / spl);  // every split non-empty
}

void csum(dpg_ctx* ctx, const float* x, int relu, const float* hw, const float* scale,
          const ConvGeom& g, float* part, int splits) {
  Params p = make_params(x, relu, hw, g);
  p.scale = scale;
  p.out = part;
  p.spl = (g.b + splits - 1) / splits;
  launch<1>(ctx, p, (unsigned)((g.b + p.spl - 1) / p.spl));
}

}  // namespace ps
}  // namespace dpg
