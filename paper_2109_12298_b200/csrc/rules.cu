// rules.cu — per-sample gradient kernels (north-star subsystem 1) with the per-sample squared
// norm fused into their epilogues (subsystem 2).
//
//   linear  : per_sample_rule_linear   (grad_sample.hpp:53-59, tensor.hpp:303-338)
//   conv2d  : per_sample_rule_conv2d   (grad_sample.hpp:135-150) with implicit im2col
//   bias    : sum_middle               (tensor.hpp:188-207), double accumulator
//   embedding: per_sample_rule_embedding (grad_sample.hpp:64-82), per-sample sorted token lists
//
// Norm partials go to a [rows, b] double slab (one row per output tile); clip_factors sums the
// rows in parameter order (optimizer.hpp:67-89).
#include "conv_common.cuh"

namespace dpg {

// ------------------------------------------------------------------------------------------
// Linear, mid == 1: G[n, o, i] = B[n, o] * A[n, i] — a single fp32 product per element, the
// same value the reference stores (0 + b*a), so this path is bit-exact. Pure store-bound:
// 128-bit streaming stores, norm accumulated in double from the stored values.
// ------------------------------------------------------------------------------------------
constexpr int kOuterChunk = 8192;  // elements of one sample's G per CTA

__global__ void __launch_bounds__(256) gs_linear_outer_kernel(const float* __restrict__ acts,
                                                              int acts_relu,
                                                              const float* __restrict__ hw,
                                                              int64_t d, int64_t r,
                                                              float* __restrict__ gw,
                                                              double* __restrict__ sq_part,
                                                              int64_t b) {
  pdl_wait();
  const int n = blockIdx.y;
  const int64_t total = r * d;
  const int64_t c0 = (int64_t)blockIdx.x * kOuterChunk;
  const int64_t c1 = c0 + kOuterChunk < total ? c0 + kOuterChunk : total;
  const float* a = acts + (int64_t)n * d;
  const float* bb = hw + (int64_t)n * r;
  float* g = gw ? gw + (int64_t)n * total : nullptr;
  double sq = 0.0;
  if ((d & 3) == 0) {
    for (int64_t e = c0 + 4 * threadIdx.x; e < c1; e += 4 * 256) {
      const int64_t o = e / d, i = e - o * d;
      const float bv = __ldg(bb + o);
      float4 av = __ldg(reinterpret_cast<const float4*>(a + i));
      av.x = relu_if(av.x, acts_relu); av.y = relu_if(av.y, acts_relu);
      av.z = relu_if(av.z, acts_relu); av.w = relu_if(av.w, acts_relu);
      const float4 v = make_float4(bv * av.x, bv * av.y, bv * av.z, bv * av.w);
      if (g) st_stream4(g + e, v);
      sq += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
  } else {
    for (int64_t e = c0 + threadIdx.x; e < c1; e += 256) {
      const int64_t o = e / d, i = e - o * d;
      const float v = __ldg(bb + o) * relu_if(__ldg(a + i), acts_relu);
      if (g) st_stream(g + e, v);
      sq += (double)v * v;
    }
  }
  __shared__ double red[8];
  const double t = block_sum<256>(sq, red);
  if (threadIdx.x == 0 && sq_part) sq_part[(int64_t)blockIdx.x * b + n] = t;
}

int sq_rows_linear(int64_t mid, int64_t d, int64_t r) {
  if (mid == 1) return (int)((r * d + kOuterChunk - 1) / kOuterChunk);
  return tc::gs_linear_rows(d, r);
}

void launch_gs_linear(dpg_ctx* ctx, const float* acts, int acts_relu, const float* hw, int64_t b,
                      int64_t mid, int64_t d, int64_t r, float* gw, double* sq_part) {
  if (b == 0) return;
  if (mid == 1) {
    dim3 grid((unsigned)((r * d + kOuterChunk - 1) / kOuterChunk), (unsigned)b);
    ::dpg::launch_pdl(gs_linear_outer_kernel, grid, 256, 0, ctx->stream, acts, acts_relu, hw, d, r, gw, sq_part, b);
    DPG_LAUNCH_CHECK(ctx);
    return;
  }
  if (tg::lin_ok(acts, hw, gw, b, mid, d, r)) {  // TMA-fed core (same norm-row order)
    tg::lin_rule(ctx, acts, acts_relu, hw, b, mid, d, r, gw, sq_part);
    return;
  }
  tc::linear_gs(ctx, acts, acts_relu, hw, b, mid, d, r, gw, sq_part);
}

// ------------------------------------------------------------------------------------------
// Conv2d: G[n, oc, k] = sum_p B[n, oc, p] * X~[n, k, p], X~ = im2col(x) gathered on the fly
// (layers.hpp:290-324 index map: k = (c*kh + ki)*kw + kj, p = oy*ow + ox).
// ------------------------------------------------------------------------------------------
int sq_rows_conv2d(const ConvGeom& g, bool nhwc_rule) {
  if (nhwc_rule) return 3;  // tg_conv.cu ConvRuleT: one partial per three-tap tile
  if (tk::supported(g)) return 1;
  if (rs::supported(g)) return rs::gs_rows(g);
  return tc::gs_conv_rows(g);
}

bool gs_conv2d_fuses_bias(const ConvGeom& g) {
  return tk::supported(g) || rs::supported(g);
}
int sq_rows_conv2d_bias(const ConvGeom& g) {
  if (tk::supported(g)) return 1;
  if (rs::supported(g)) return rs::gs_rows(g);
  return 1;
}

void launch_gs_conv2d(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const ConvGeom& g,
                      float* gw, double* sq_part, float* gb, double* sq_b, bool hw_nhwc, const float* xh) {
  if (g.b == 0) return;
  const bool bias = gb || sq_b;
  if (xh) {  // the layer input's NHWC copy exists: the TMA-fed core (tg_conv.cu ConvRuleT)
    if (hw_nhwc || !tg::rule_nhwc_ok(g)) raise(DPG_ERR_INTERNAL, "NHWC conv rule: unsupported geometry");
    if (bias) launch_gs_bias(ctx, hw, g.b, g.P(), g.oc, true, gb, sq_b);
    tg::conv_rule_nhwc(ctx, xh, hw, g, gw, sq_part);
    return;
  }
  if (tk::supported(g)) {
    tk::gs(ctx, x, x_relu, hw, g, gw, sq_part, gb, sq_b, hw_nhwc);
    return;
  }
  if (hw_nhwc) raise(DPG_ERR_INTERNAL, "channels-last highway needs the thin-K rule");
  if (rs::supported(g)) {
    rs::gs(ctx, x, x_relu, hw, g, gw, sq_part, gb, sq_b);
    return;
  }
  if (bias) launch_gs_bias(ctx, hw, g.b, g.P(), g.oc, true, gb, sq_b);
  tc::conv_gs(ctx, x, x_relu, hw, g, gw, sq_part);
}

// ------------------------------------------------------------------------------------------
// Bias: gb[n, o] = (float) sum_mid (double) hw (sum_middle, tensor.hpp:197-205). Conv layout:
// one warp per row with a fixed fp64 tree; linear layout [mid][r]: sequential in mid, coalesced
// over o. One CTA per sample; norm partial = one row.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 4) gs_bias_kernel(const float* __restrict__ hw, int64_t mid,
                                                      int64_t r, int conv_layout,
                                                      float* __restrict__ gb,
                                                      double* __restrict__ sq_part, int64_t b) {
  pdl_wait();
  const int64_t n = blockIdx.x;
  double sq = 0.0;
  if (conv_layout) {
    // rows [r][mid] of sample n are contiguous: one warp per row, lanes take strided elements,
    // fp64 partials combined by a fixed shuffle tree (a different association of the same fp64
    // sum than the reference's sequential loop: the float result agrees to the last bit except
    // in rare rounding-boundary cases, within the 1e-7 bias tolerance)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t o = warp;
    if (mid <= 64) {
      // short rows (e.g. an 8x8 feature map): 8 rows per warp, all 16 loads issued first and the
      // 8 shuffle trees interleaved (same association as below)
      constexpr int RW = 8;
      for (; o < r; o += 8 * RW) {
        float v[RW][2];
#pragma unroll
        for (int q = 0; q < RW; ++q)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int64_t m = lane + 32 * i, oq = o + 8 * q;
            v[q][i] = (oq < r && m < mid) ? __ldg(hw + (n * r + oq) * mid + m) : 0.f;
          }
        double acc[RW];
#pragma unroll
        for (int q = 0; q < RW; ++q) {
          acc[q] = 0.0;
#pragma unroll
          for (int i = 0; i < 2; ++i)
            if (lane + 32 * i < mid) acc[q] += (double)v[q][i];
        }
#pragma unroll
        for (int q = 0; q < RW; ++q) acc[q] = warp_sum(acc[q]);
#pragma unroll
        for (int q = 0; q < RW; ++q) {
          const int64_t oq = o + 8 * q;
          const float fv = (float)acc[q];
          if (lane == 0 && oq < r) {
            if (gb) gb[n * r + oq] = fv;
            sq += (double)fv * fv;
          }
        }
      }
    } else if (mid <= 256) {
      // 4 rows at a time, every lane's loads issued before the sums (same association)
      for (; o + 24 < r; o += 32) {
        float v[4][8];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int64_t m = lane + 32 * i;
            v[q][i] = m < mid ? __ldg(hw + (n * r + o + 8 * q) * mid + m) : 0.f;
          }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (lane + 32 * i < mid) acc += (double)v[q][i];
          acc = warp_sum(acc);
          const float fv = (float)acc;
          if (lane == 0) {
            if (gb) gb[n * r + o + 8 * q] = fv;
            sq += (double)fv * fv;
          }
        }
      }
    }
    for (; o < r; o += 8) {
      const float* row = hw + (n * r + o) * mid;
      double acc = 0.0;
#pragma unroll 8
      for (int64_t m = lane; m < mid; m += 32) acc += (double)__ldg(row + m);
      acc = warp_sum(acc);
      const float v = (float)acc;
      if (lane == 0) {
        if (gb) gb[n * r + o] = v;
        sq += (double)v * v;
      }
    }
  } else if (r % 4 == 0 && (reinterpret_cast<uintptr_t>(hw) & 15) == 0) {
    // 4 consecutive outputs per thread: 16 float4 loads in flight, each column summed in order
    for (int64_t o = 4 * (int64_t)threadIdx.x; o < r; o += 4 * 256) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const float* col = hw + n * mid * r + o;
      int64_t m = 0;
      for (; m + 16 <= mid; m += 16) {
        float4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(col + (m + u) * r));
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          a0 += (double)v[u].x; a1 += (double)v[u].y; a2 += (double)v[u].z; a3 += (double)v[u].w;
        }
      }
      for (; m < mid; ++m) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(col + m * r));
        a0 += (double)v.x; a1 += (double)v.y; a2 += (double)v.z; a3 += (double)v.w;
      }
      const float f[4] = {(float)a0, (float)a1, (float)a2, (float)a3};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (gb) gb[n * r + o + e] = f[e];
        sq += (double)f[e] * f[e];
      }
    }
  } else {
    for (int64_t o = threadIdx.x; o < r; o += 256) {
      double acc = 0.0;
      const float* col = hw + n * mid * r + o;
      int64_t m = 0;
      for (; m + 16 <= mid; m += 16) {  // 16 loads in flight, summed in order
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldg(col + (m + u) * r);
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += (double)v[u];
      }
      for (; m < mid; ++m) acc += (double)__ldg(col + m * r);
      const float v = (float)acc;
      if (gb) gb[n * r + o] = v;
      sq += (double)v * v;
    }
  }
  __shared__ double red[8];
  const double t = block_sum<256>(sq, red);
  if (threadIdx.x == 0 && sq_part) sq_part[n] = t;
}

void launch_gs_bias(dpg_ctx* ctx, const float* hw, int64_t b, int64_t mid, int64_t r,
                    bool hw_layout_conv, float* gb, double* sq_part) {
  if (b == 0) return;
  ::dpg::launch_pdl(gs_bias_kernel, (unsigned)b, 256, 0, ctx->stream, hw, mid, r, hw_layout_conv ? 1 : 0, gb, sq_part, b);
  DPG_LAUNCH_CHECK(ctx);
}

// ------------------------------------------------------------------------------------------
// Embedding. Step 1: per-sample stable sort of the token ids (key = v * 2^32 + s), validating
// each id as require_integral_index does (layers.hpp:368-376). Invalid ids report
// (stage EMBED_INDEX, sample-major position n*t+s) and are clamped to 0.
// ------------------------------------------------------------------------------------------
constexpr int kSortThreads = 512;
constexpr int kMaxTokens = 4096;

__global__ void __launch_bounds__(kSortThreads) embed_sort_kernel(const float* __restrict__ idx,
                                                                  int64_t t, int64_t vocab,
                                                                  int32_t* __restrict__ sorted_v,
                                                                  int32_t* __restrict__ sorted_s,
                                                                  DeviceErr* err) {
  pdl_wait();
  __shared__ unsigned long long keys[kMaxTokens];
  const int64_t n = blockIdx.x;
  int p2 = 1;
  while (p2 < t) p2 <<= 1;
  for (int s = threadIdx.x; s < p2; s += kSortThreads) {
    unsigned long long key = ~0ull;
    if (s < t) {
      const float raw = __ldg(idx + n * t + s);
      const double v = (double)raw;
      uint32_t vi = 0;
      if (!(v >= 0.0) || v != floor(v) || v >= (double)vocab) {
        report_error(err, err_key(ERR_STAGE_EMBED_INDEX, 0, (uint64_t)(n * t + s)),
                     (uint64_t)__float_as_uint(raw));
      } else {
        vi = (uint32_t)v;
      }
      key = ((unsigned long long)vi << 32) | (unsigned long long)s;
    }
    keys[s] = key;
  }
  __syncthreads();
  // bitonic sort, ascending
  for (int k = 2; k <= p2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < p2; i += kSortThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long a = keys[i], c = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > c) == up) {
            keys[i] = c;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int s = threadIdx.x; s < t; s += kSortThreads) {
    sorted_v[n * t + s] = (int32_t)(keys[s] >> 32);
    sorted_s[n * t + s] = (int32_t)(keys[s] & 0xFFFFFFFFull);
  }
}

void launch_embed_sort(dpg_ctx* ctx, const float* idx, int64_t b, int64_t t, int64_t vocab,
                       int32_t* sorted_v, int32_t* sorted_s) {
  if (t > kMaxTokens) raise(DPG_ERR_DIMENSION, "embedding: at most 4096 tokens per sample on device");
  if (b == 0 || t == 0) return;
  ::dpg::launch_pdl(embed_sort_kernel, (unsigned)b, kSortThreads, 0, ctx->stream, idx, t, vocab, sorted_v, sorted_s, ctx->dev_err);
  DPG_LAUNCH_CHECK(ctx);
}

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Step 2 (dense): each CTA owns kEmbRows consecutive rows of one sample's [vocab, dim] gradient
// (one contiguous block). The block is first zero-filled with coalesced 128-bit streaming
// stores — >97 % of the record is zeros (a sample touches at most t of the vocab rows) — then
// the rows the sample's tokens hit are overwritten with their sums over duplicates in ascending
// s (grad_sample.hpp:75-79), in the same CTA after a barrier.
constexpr int kEmbRows = 64;

__global__ void __launch_bounds__(256) gs_embedding_dense_kernel(
    const int32_t* __restrict__ sorted_v, const int32_t* __restrict__ sorted_s,
    const float* __restrict__ hw, int64_t t, int64_t vocab, int64_t dim, float* __restrict__ g,
    double* __restrict__ sq_part, int64_t b) {
  pdl_wait();
  extern __shared__ int32_t sv[];
  __shared__ int range[2];
  const int64_t n = blockIdx.y;
  const int64_t v0 = (int64_t)blockIdx.x * kEmbRows;
  const int64_t nrows = vocab - v0 < kEmbRows ? vocab - v0 : kEmbRows;
  float* blk = g + (n * vocab + v0) * dim;
  const int64_t total = nrows * dim;
  if ((dim & 3) == 0) {
    float4* b4 = reinterpret_cast<float4*>(blk);
    for (int64_t i = threadIdx.x; i < total / 4; i += 256) st_stream4(reinterpret_cast<float*>(b4 + i), make_float4(0.f, 0.f, 0.f, 0.f));
  } else {
    for (int64_t i = threadIdx.x; i < total; i += 256) st_stream(blk + i, 0.f);
  }
  for (int s = threadIdx.x; s < t; s += 256) sv[s] = sorted_v[n * t + s];
  __syncthreads();
  if (threadIdx.x < 2) range[threadIdx.x] = lower_bound_i32(sv, (int)t, (int32_t)(v0 + (threadIdx.x ? nrows : 0)));
  __syncthreads();  // also orders the zero fill before the row writes below
  const int lo = range[0], hi = range[1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* ss = sorted_s + n * t;
  const float* hwn = hw + n * t * dim;
  double sq = 0.0;
  int r = 0;  // run index: warp w takes runs w, w + 8, ...
  for (int j0 = lo; j0 < hi; ++r) {
    int j1 = j0 + 1;
    while (j1 < hi && sv[j1] == sv[j0]) ++j1;
    if ((r & 7) == warp) {
      float* row = g + (n * vocab + sv[j0]) * dim;
      if ((dim & 3) == 0) {
        for (int64_t d0 = 4 * lane; d0 < dim; d0 += 128) {
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int j = j0; j < j1; ++j) {
            const float4 h = __ldg(reinterpret_cast<const float4*>(hwn + (int64_t)ss[j] * dim + d0));
            acc.x += h.x; acc.y += h.y; acc.z += h.z; acc.w += h.w;
          }
          st_stream4(row + d0, acc);
          sq += (double)acc.x * acc.x + (double)acc.y * acc.y + (double)acc.z * acc.z + (double)acc.w * acc.w;
        }
      } else {
        for (int64_t d0 = lane; d0 < dim; d0 += 32) {
          float acc = 0.f;
          for (int j = j0; j < j1; ++j) acc += __ldg(hwn + (int64_t)ss[j] * dim + d0);
          st_stream(row + d0, acc);
          sq += (double)acc * acc;
        }
      }
    }
    j0 = j1;
  }
  __shared__ double red[8];
  const double tot = block_sum<256>(sq, red);
  if (threadIdx.x == 0 && sq_part) sq_part[(int64_t)blockIdx.x * b + n] = tot;
}

// Step 2 (sparse): norms only — one CTA per sample walks its unique ids.
__global__ void __launch_bounds__(256) gs_embedding_sq_kernel(
    const int32_t* __restrict__ sorted_v, const int32_t* __restrict__ sorted_s,
    const float* __restrict__ hw, int64_t t, int64_t dim, double* __restrict__ sq_part) {
  pdl_wait();
  const int64_t n = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* sv = sorted_v + n * t;
  const int32_t* ss = sorted_s + n * t;
  const float* hwn = hw + n * t * dim;
  double sq = 0.0;
  for (int64_t j0 = warp; j0 < t; j0 += 8) {
    if (j0 > 0 && sv[j0] == sv[j0 - 1]) continue;  // not a segment start
    int64_t hi = j0;
    while (hi < t && sv[hi] == sv[j0]) ++hi;
    for (int64_t d0 = lane; d0 < dim; d0 += 32) {
      float acc = 0.f;
      for (int64_t j = j0; j < hi; ++j) acc += __ldg(hwn + (int64_t)ss[j] * dim + d0);
      sq += (double)acc * acc;
    }
  }
  __shared__ double red[8];
  const double tot = block_sum<256>(sq, red);
  if (threadIdx.x == 0) sq_part[n] = tot;
}

int sq_rows_embedding(int64_t vocab, int64_t dim) {
  (void)dim;
  return (int)((vocab + kEmbRows - 1) / kEmbRows);
}

void launch_gs_embedding(dpg_ctx* ctx, const int32_t* sorted_v, const int32_t* sorted_s,
                         const float* hw, int64_t b, int64_t t, int64_t vocab, int64_t dim,
                         float* g, double* sq_part) {
  if (b == 0) return;
  if (g) {
    dim3 grid((unsigned)((vocab + kEmbRows - 1) / kEmbRows), (unsigned)b);
    ::dpg::launch_pdl(gs_embedding_dense_kernel, grid, 256, sizeof(int32_t) * t, ctx->stream, 
        sorted_v, sorted_s, hw, t, vocab, dim, g, sq_part, b);
  } else {
    // sparse mode: the norm lands in the first row; the remaining rows are zero-filled so the
    // slab layout does not depend on the mode
    const int rows = sq_rows_embedding(vocab, dim);
    if (rows > 1) DPG_CUDA(cudaMemsetAsync(sq_part + b, 0, sizeof(double) * (size_t)(rows - 1) * b, ctx->stream));
    ::dpg::launch_pdl(gs_embedding_sq_kernel, (unsigned)b, 256, 0, ctx->stream, sorted_v, sorted_s, hw, t, dim, sq_part);
  }
  DPG_LAUNCH_CHECK(ctx);
}

// ------------------------------------------------------------------------------------------
__global__ void sq_reduce_kernel(const double* __restrict__ part, int rows, int64_t b,
                                 double* __restrict__ out) {
  pdl_wait();
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= b) return;
  double acc = 0.0;
  for (int r = 0; r < rows; ++r) acc += part[(int64_t)r * b + n];
  out[n] = acc;
}

void launch_sq_reduce(dpg_ctx* ctx, const double* part, int rows, int64_t b, double* out) {
  if (b == 0) return;
  ::dpg::launch_pdl(sq_reduce_kernel, (unsigned)((b + 255) / 256), 256, 0, ctx->stream, part, rows, b, out);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace dpg
