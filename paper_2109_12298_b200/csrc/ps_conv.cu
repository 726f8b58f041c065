// ps_conv.cu — per-sample conv contractions with the sample staged in shared memory.
//
//   GS   : G[n][oc][kcol] = sum_p B[n, oc, p] X~[n, kcol, p]   (per_sample_rule_conv2d,
//          grad_sample.hpp:135-150) + the fused ||G_n||^2 partial
//   CSUM : S[oc][kcol]    = sum_n s_n sum_p B[n, oc, p] X~[n, kcol, p]   (clip_and_sum pass 2,
//          optimizer.hpp:99-114, without materialising G)
//
// One CTA owns an oc tile and one sample (GS) or a contiguous group of samples (CSUM). For each
// sample it stages x_n (the whole input image, 128-bit loads) and the highway rows of its oc tile
// in shared memory, expands im2col into shared memory one chunk of positions at a time
// (X~ stored [p][kcol] so four consecutive kcol are one 128-bit read), and every thread
// accumulates a 4 (kcol) x 8 (oc) register block over p. GS writes each block with 128-bit
// streaming stores — the per-sample gradient is the dominant HBM stream of the step, written
// exactly once. CSUM keeps its register blocks across the group's samples (weighted by s_n) and
// writes one partial per CTA for the fixed-order split reduce.
//
// These shapes (P = positions per sample <= 256, a few thousand outputs per sample) are
// store- or latency-bound, not tensor-bound: CUDA cores with shared-memory reuse beat a tensor
// tile padded from K = P to 32 (kernel table).
#include <cstdlib>

#include "conv_common.cuh"

namespace dpg {
namespace ps {

constexpr int kThreads = 256;
constexpr int kPChunk = 16;

struct Params {
  const float* x;
  int relu;
  const float* hw;
  const float* scale;  // CSUM
  float* out;          // GS: G [b, oc, Kc]; CSUM: partials [splits, oc, Kc]
  double* sq_part;     // GS: [oc_tiles, b]
  int64_t b, spl;
  int ic, h, w, oc, kh, kw, stride, pad, oh, ow, P, Kc, Kc4, oct;
};

template <int MODE, int OCT, int ITEMS>
__global__ void __launch_bounds__(kThreads) ps_conv_kernel(const Params p) {
  extern __shared__ float sm[];
  const int hwsz = p.ic * p.h * p.w;
  float* xs = sm;                                  // [ic*h*w]
  float* hs = xs + ((hwsz + 3) & ~3);              // [P][OCT]
  float* xt = hs + p.P * OCT;                      // [kPChunk][Kc4]
  int* kt = reinterpret_cast<int*>(xt + kPChunk * p.Kc4);  // [Kc4]: packed (c*h*w, ki, kj)
  const int tid = threadIdx.x;
  const int oc0 = blockIdx.x * OCT;
  const int n_begin = (int)(MODE == 0 ? blockIdx.y : blockIdx.y * p.spl);
  const int n_end = (int)(MODE == 0 ? blockIdx.y + 1 : min((int64_t)(blockIdx.y + 1) * p.spl, p.b));
  const int nq = p.Kc4 / 4;           // kcol quads
  const int ngrp = OCT / 8;           // oc groups of 8
  const int nitems = nq * ngrp;

  for (int k = tid; k < p.Kc4; k += kThreads) {
    int e = -1;
    if (k < p.Kc) {
      const int khw = p.kh * p.kw;
      const int c = k / khw, r = k - c * khw;
      const int ki = r / p.kw, kj = r - ki * p.kw;
      e = (c << 10) | (ki << 5) | kj;  // ic < 2^21, kh, kw < 32
    }
    kt[k] = e;
  }

  float acc[ITEMS][8][4];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[it][i][j] = 0.f;
  double sq = 0.0;

  for (int n = n_begin; n < n_end; ++n) {
    __syncthreads();  // previous sample fully consumed
    // stage x_n and the oc tile of B_n (scaled by s_n in CSUM mode)
    const float* xn = p.x + (int64_t)n * hwsz;
    if ((hwsz & 3) == 0) {
      for (int i = tid; i < hwsz / 4; i += kThreads) {
        float4 v = __ldg(reinterpret_cast<const float4*>(xn) + i);
        v.x = relu_if(v.x, p.relu); v.y = relu_if(v.y, p.relu);
        v.z = relu_if(v.z, p.relu); v.w = relu_if(v.w, p.relu);
        reinterpret_cast<float4*>(xs)[i] = v;
      }
    } else {
      for (int i = tid; i < hwsz; i += kThreads) xs[i] = relu_if(__ldg(xn + i), p.relu);
    }
    const float sn = MODE == 1 ? __ldg(p.scale + n) : 1.f;
    for (int i = tid; i < OCT * p.P; i += kThreads) {
      const int q = i / OCT, o = i - q * OCT;  // conflict-free transposed store; rows hit L1
      float v = 0.f;
      if (oc0 + o < p.oc) v = __ldg(p.hw + ((int64_t)n * p.oc + oc0 + o) * p.P + q);
      hs[q * OCT + o] = MODE == 1 ? sn * v : v;
    }
    for (int p0 = 0; p0 < p.P; p0 += kPChunk) {
      const int pc = min(kPChunk, p.P - p0);
      __syncthreads();  // staging done / previous chunk consumed
      for (int i = tid; i < pc * p.Kc4; i += kThreads) {
        const int pp = i / p.Kc4, k = i - pp * p.Kc4;
        const int e = kt[k];
        float v = 0.f;
        if (e >= 0) {
          const int pos = p0 + pp;
          const int oy = pos / p.ow, ox = pos - oy * p.ow;
          const int iy = oy * p.stride + ((e >> 5) & 31) - p.pad;
          const int ix = ox * p.stride + (e & 31) - p.pad;
          if ((unsigned)iy < (unsigned)p.h && (unsigned)ix < (unsigned)p.w)
            v = xs[((e >> 10) * p.h + iy) * p.w + ix];
        }
        xt[pp * p.Kc4 + k] = v;
      }
      __syncthreads();
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) {
        const int item = tid + it * kThreads;
        if (item < nitems) {
          const int q4 = item % nq, g = item / nq;
          for (int pp = 0; pp < pc; ++pp) {
            const float4 xv = *reinterpret_cast<const float4*>(xt + pp * p.Kc4 + 4 * q4);
            const float4 h0 = *reinterpret_cast<const float4*>(hs + (p0 + pp) * OCT + 8 * g);
            const float4 h1 = *reinterpret_cast<const float4*>(hs + (p0 + pp) * OCT + 8 * g + 4);
            const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              acc[it][i][0] = fmaf(hv[i], xv.x, acc[it][i][0]);
              acc[it][i][1] = fmaf(hv[i], xv.y, acc[it][i][1]);
              acc[it][i][2] = fmaf(hv[i], xv.z, acc[it][i][2]);
              acc[it][i][3] = fmaf(hv[i], xv.w, acc[it][i][3]);
            }
          }
        }
      }
    }
    if (MODE == 0) {
      // write G_n blocks, accumulate the norm, reset for the next sample (none in GS mode)
#pragma unroll
      for (int it = 0; it < ITEMS; ++it) {
        const int item = tid + it * kThreads;
        if (item < nitems) {
          const int q4 = item % nq, g = item / nq;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int oc = oc0 + 8 * g + i;
            if (oc < p.oc) {
              float* row = p.out ? p.out + ((int64_t)n * p.oc + oc) * p.Kc : nullptr;
              const int k0 = 4 * q4;
              if (row && (p.Kc & 3) == 0) {
                st_stream4(row + k0, make_float4(acc[it][i][0], acc[it][i][1], acc[it][i][2], acc[it][i][3]));
              } else if (row) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  if (k0 + j < p.Kc) st_stream(row + k0 + j, acc[it][i][j]);
              }
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (k0 + j < p.Kc) sq += (double)acc[it][i][j] * acc[it][i][j];
            }
          }
        }
      }
    }
  }
  if (MODE == 1) {
    float* base = p.out + (int64_t)blockIdx.y * p.oc * p.Kc;
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int item = tid + it * kThreads;
      if (item < nitems) {
        const int q4 = item % nq, g = item / nq;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int oc = oc0 + 8 * g + i;
          if (oc < p.oc) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (4 * q4 + j < p.Kc) base[(int64_t)oc * p.Kc + 4 * q4 + j] = acc[it][i][j];
          }
        }
      }
    }
  } else {
    __shared__ double red[kThreads / 32];
    const double t = block_sum<kThreads>(sq, red);
    if (tid == 0 && p.sq_part) p.sq_part[(int64_t)blockIdx.x * p.b + blockIdx.y] = t;
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
  return p;
}

inline size_t smem_bytes(const Params& p, int oct) {
  const int hwsz = p.ic * p.h * p.w;
  return sizeof(float) * (size_t)(((hwsz + 3) & ~3) + p.P * oct + kPChunk * p.Kc4) + sizeof(int) * p.Kc4;
}

// usable when one sample's image, its highway tile and a position chunk fit in shared memory
// shape check only (shared memory fits, kernel index packing)
bool fits(const ConvGeom& g) {
  Params p = make_params(nullptr, 0, nullptr, g);
  const int nitems_gs = (p.Kc4 / 4) * (32 / 8);
  return g.kh < 32 && g.kw < 32 && nitems_gs <= 3 * kThreads && smem_bytes(p, 32) <= 200 * 1024;
}

// Per-sample gradients of layers with few positions per sample (P <= 16) are store-bound: the
// staged CUDA-core kernel streams G faster than a tensor tile padded from K = P to 32
// (measured on B200). Larger P and the clipped sums go to tcgen05.
// DPG_PS=0 / DPG_PS=1 force it off / on for A/B measurements.
bool supported(const ConvGeom& g) {
  static const int force = [] {
    const char* e = std::getenv("DPG_PS");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  if (!fits(g) || force == 0) return false;
  return force == 1 || g.P() <= 16;
}
bool supported_csum(const ConvGeom& g) {
  static const bool force = [] {
    const char* e = std::getenv("DPG_PS");
    return e && e[0] == '1';
  }();
  return force && fits(g);
}

template <int MODE, int OCT>
static void launch(dpg_ctx* ctx, const Params& p, unsigned gy) {
  const size_t smem = smem_bytes(p, OCT);
  const int nitems = (p.Kc4 / 4) * (OCT / 8);
  const int items = (nitems + kThreads - 1) / kThreads;
  dim3 grid((unsigned)((p.oc + OCT - 1) / OCT), gy);
  auto go = [&](auto kern) {
    static int attr = 0;
    if ((int)smem > attr) {
      DPG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = (int)smem;
    }
    kern<<<grid, kThreads, smem, ctx->stream>>>(p);
  };
  if (items <= 1) go(ps_conv_kernel<MODE, OCT, 1>);
  else if (items <= 2) go(ps_conv_kernel<MODE, OCT, 2>);
  else if (items <= 3) go(ps_conv_kernel<MODE, OCT, 3>);
  else raise(DPG_ERR_INTERNAL, "ps_conv: tile too large");
  DPG_LAUNCH_CHECK(ctx);
}

constexpr int kGsOct = 32;
constexpr int kCsOct = 16;

int gs_rows(const ConvGeom& g) { return (int)((g.oc + kGsOct - 1) / kGsOct); }

void gs(dpg_ctx* ctx, const float* x, int relu, const float* hw, const ConvGeom& g, float* gw,
        double* sq_part) {
  Params p = make_params(x, relu, hw, g);
  p.out = gw;
  p.sq_part = sq_part;
  // items per thread: (Kc4/4) * 4 groups <= 768 for Kc <= 768
  launch<0, kGsOct>(ctx, p, (unsigned)g.b);
}

int csum_splits(const ConvGeom& g) {
  const int64_t tiles = (g.oc + kCsOct - 1) / kCsOct;
  int64_t splits = (2 * kNumSMs + tiles - 1) / tiles;
  return (int)std::max<int64_t>(1, std::min<int64_t>(splits, g.b));
}

void csum(dpg_ctx* ctx, const float* x, int relu, const float* hw, const float* scale,
          const ConvGeom& g, float* part, int splits) {
  Params p = make_params(x, relu, hw, g);
  p.scale = scale;
  p.out = part;
  p.spl = (g.b + splits - 1) / splits;
  launch<1, kCsOct>(ctx, p, (unsigned)splits);
}

}  // namespace ps
}  // namespace dpg
