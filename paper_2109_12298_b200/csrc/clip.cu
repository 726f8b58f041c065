// clip.cu — clip factors and clipped sums (north-star subsystems 2-3).
//
//   clip_factors : clip_and_sum pass 1 tail + factors (optimizer.hpp:67-98)
//   clipped sums : clip_and_sum pass 2 (optimizer.hpp:99-114) formed as (scale ⊙ B)^T A from the
//                  activations and highway gradients — the materialised per-sample gradients are
//                  not read again. Split-K over samples with a fixed-order reduction, so results
//                  are deterministic and identical on every replay.
//   materialised : the reference's own pass 2 over a stored record, in its exact order.
#include "conv_common.cuh"

namespace dpg {

// ------------------------------------------------------------------------------------------
// Clip factors. slab [rows, b]: per-(parameter tile, sample) squared norms; row_param[r] is the
// parameter index owning row r (rows are in parameter order). Sum rows in order, flag the first
// non-finite parameter per sample (NumericError, optimizer.hpp:77-83), then
// norm = sqrt(sq), scale = (float)(C / max(norm, C)), count norm > C.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) clip_factors_kernel(const double* __restrict__ slab,
                                                           const int32_t* __restrict__ row_param,
                                                           int rows, int64_t b, double c,
                                                           double* __restrict__ norms,
                                                           float* __restrict__ scale,
                                                           unsigned long long* num_clipped,
                                                           DeviceErr* err, unsigned long long* sync) {
  pdl_wait();
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int clipped = 0;
  if (n < b) {
    double sq = 0.0;
    int bad = -1;
    // every row's load of a 32-row batch issued before the in-order sum (a short tail of rows
    // must not become a chain of dependent loads)
    for (int r = 0; r < rows; r += 32) {
      double v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = r + u < rows ? slab[(int64_t)(r + u) * b + n] : 0.0;
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        if (r + u >= rows) break;
        if (bad < 0 && !isfinite(v[u])) bad = row_param ? row_param[r + u] : 0;
        sq += v[u];
      }
    }
    if (bad >= 0) report_error(err, err_key(ERR_STAGE_NONFINITE, (uint64_t)bad, (uint64_t)n), 0);
    const double norm = sqrt(sq);
    const double s = c / (norm < c ? c : norm);  // C / std::max(norm, C)
    if (norms) norms[n] = norm;
    scale[n] = (float)s;
    clipped = norm > c ? 1 : 0;
  }
  // num_clipped without a memset launch before the kernel: CTAs add into a context accumulator;
  // the last CTA to take a ticket publishes the total and resets the accumulator and the ticket
  const int cnt = __syncthreads_count(clipped);
  if (threadIdx.x == 0 && num_clipped) {
    if (cnt) atomicAdd(&sync[0], (unsigned long long)cnt);
    __threadfence();
    if (atomicAdd(&sync[1], 1ull) == gridDim.x - 1) {
      __threadfence();
      *num_clipped = atomicExch(&sync[0], 0ull);
      atomicExch(&sync[1], 0ull);
    }
  }
}

void launch_clip_factors(dpg_ctx* ctx, const double* slab, const int32_t* row_param, int rows,
                         int64_t b, double c, double* norms, float* scale, int64_t* num_clipped) {
  if (b == 0) {
    if (num_clipped) DPG_CUDA(cudaMemsetAsync(num_clipped, 0, sizeof(int64_t), ctx->stream));
    return;
  }
  ::dpg::launch_pdl(clip_factors_kernel, (unsigned)((b + 63) / 64), 64, 0, ctx->stream, 
      slab, row_param, rows, b, c, norms, scale, reinterpret_cast<unsigned long long*>(num_clipped),
      ctx->dev_err, ctx->clip_sync);
  DPG_LAUNCH_CHECK(ctx);
}

// ------------------------------------------------------------------------------------------
// Column sums over a leading index z (samples or split-K partials):
//   out[j] = [out[j] +] sum_z c(z) v(z, j)
// A CTA owns 32 consecutive columns (lanes) and splits z into kColWarps contiguous ranges, one per
// warp; each warp keeps kColBatch loads in flight and the warp partials are combined in warp order,
// so the result is deterministic (identical on every run and replay).
// ------------------------------------------------------------------------------------------
constexpr int kColWarps = 16;
constexpr int kColBatch = 16;

struct IdOut {
  __device__ __forceinline__ int64_t operator()(int64_t j) const { return j; }
};

template <class V, class C, class OI = IdOut>
__device__ __forceinline__ void colsum_body(const V& v, const C& c, int64_t nz, int64_t ncol,
                                            int64_t j0, float* __restrict__ out, int accumulate,
                                            OI oi = IdOut{}) {
  __shared__ float part[kColWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = j0 + lane;
  const int64_t z0 = nz * warp / kColWarps, z1 = nz * (warp + 1) / kColWarps;
  float acc = 0.f;
  if (j < ncol) {
    int64_t z = z0;
    for (; z + kColBatch <= z1; z += kColBatch) {
      float vv[kColBatch], cc[kColBatch];
#pragma unroll
      for (int u = 0; u < kColBatch; ++u) {
        vv[u] = v(z + u, j);
        cc[u] = c(z + u);
      }
#pragma unroll
      for (int u = 0; u < kColBatch; ++u) acc = fmaf(cc[u], vv[u], acc);
    }
    for (; z < z1; ++z) acc = fmaf(c(z), v(z, j), acc);
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && j < ncol) {
    float t = part[0][lane];
#pragma unroll
    for (int w = 1; w < kColWarps; ++w) t += part[w][lane];
    const int64_t jo = oi(j);
    out[jo] = accumulate ? out[jo] + t : t;
  }
}

struct PartV {  // split-K partials: v(z, j) = part[z * zstride + j]
  const float* part;
  int64_t zstride;
  __device__ __forceinline__ float operator()(int64_t z, int64_t j) const { return __ldg(part + z * zstride + j); }
};
struct OneC {
  __device__ __forceinline__ float operator()(int64_t) const { return 1.f; }
};
struct ScaleC {
  const float* scale;
  __device__ __forceinline__ float operator()(int64_t n) const { return __ldg(scale + n); }
};

__global__ void __launch_bounds__(32 * kColWarps) splitk_reduce_kernel(PartV v, int splits, int64_t n,
                                                                       float* out, int accumulate) {
  pdl_wait();
  colsum_body(v, OneC{}, splits, n, (int64_t)blockIdx.x * 32, out, accumulate);
}

// Split-K partials, 16-byte columns: a CTA owns 128 x 4 consecutive columns (one float4 per lane);
// its 8 warps take contiguous z ranges (kColBatch loads in flight per thread) and the warp partials
// are added in warp order — deterministic, and 4x the bytes per load of colsum_body, which left
// the wide reduces (e.g. 37 splits x 262,144 columns) latency-bound at ~1 TB/s.
constexpr int kRed4Warps = 8;
template <class OI>
__global__ void __launch_bounds__(32 * kRed4Warps) splitk_reduce4_kernel(const float* __restrict__ part, int splits,
                                                                         int64_t n, float* __restrict__ out,
                                                                         int accumulate, OI oi) {
  pdl_wait();
  __shared__ float4 red[kRed4Warps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = ((int64_t)blockIdx.x * 32 + lane) * 4;
  const int z0 = (int)((int64_t)splits * warp / kRed4Warps), z1 = (int)((int64_t)splits * (warp + 1) / kRed4Warps);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j < n) {
    const float4* p = reinterpret_cast<const float4*>(part + j);
    const int64_t zs = n / 4;
    int z = z0;
    for (; z + kColBatch <= z1; z += kColBatch) {
      float4 v[kColBatch];
#pragma unroll
      for (int u = 0; u < kColBatch; ++u) v[u] = __ldg(p + (z + u) * zs);
#pragma unroll
      for (int u = 0; u < kColBatch; ++u) {
        acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
      }
    }
    for (; z < z1; ++z) {
      const float4 v = __ldg(p + z * zs);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && j < n) {
    float4 t = red[0][lane];
#pragma unroll
    for (int w = 1; w < kRed4Warps; ++w) {
      const float4 v = red[w][lane];
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t jo = oi(j + e);
      out[jo] = accumulate ? out[jo] + tv[e] : tv[e];
    }
  }
}

template <class OI>
static bool launch_splitk_reduce4(dpg_ctx* ctx, const float* part, int splits, int64_t n, float* out,
                                  int accumulate, OI oi) {
  if (n % 4 != 0 || (reinterpret_cast<uintptr_t>(part) & 15) != 0) return false;
  ::dpg::launch_pdl(splitk_reduce4_kernel<OI>, (unsigned)((n / 4 + 31) / 32), 32 * kRed4Warps, 0, ctx->stream, part,
                    splits, n, out, accumulate, oi);
  DPG_LAUNCH_CHECK(ctx);
  return true;
}

static void launch_splitk_reduce(dpg_ctx* ctx, const float* part, int splits, int64_t n, float* out,
                                 int accumulate) {
  if (launch_splitk_reduce4(ctx, part, splits, n, out, accumulate, IdOut{})) return;
  ::dpg::launch_pdl(splitk_reduce_kernel, (unsigned)((n + 31) / 32), 32 * kColWarps, 0, ctx->stream, 
      PartV{part, n}, splits, n, out, accumulate);
  DPG_LAUNCH_CHECK(ctx);
}

// partials of the TMA-fed conv clipped sum are [split][o][(tap, channel)]: the column of the
// reference's k order (channel-major, layers.hpp:290-324) is c * khw + t
struct TapMajorOut {
  int C, khw;
  int64_t K;
  __device__ __forceinline__ int64_t operator()(int64_t j) const {
    const int64_t o = j / K, r = j - o * K, t = r / C, c = r - t * C;
    return o * K + c * khw + t;
  }
};

__global__ void __launch_bounds__(32 * kColWarps) splitk_reduce_tap_kernel(PartV v, int splits, int64_t n,
                                                                           float* out, int accumulate,
                                                                           TapMajorOut oi) {
  pdl_wait();
  colsum_body(v, OneC{}, splits, n, (int64_t)blockIdx.x * 32, out, accumulate, oi);
}

// ------------------------------------------------------------------------------------------
// Weighted sums over samples with few outputs: out[j] (+)= sum_n s_n v(n, j) (colsum_body).
// ------------------------------------------------------------------------------------------
struct OuterV {  // linear, mid == 1: v(n, o*d + i) = B[n, o] * A[n, i]
  const float* acts;
  const float* hw;
  int64_t d, r;
  int relu;
  __device__ __forceinline__ float operator()(int64_t n, int64_t j) const {
    const int64_t o = (uint32_t)j / (uint32_t)d, i = j - o * d;  // d * r < 2^31 (launch check)
    return __ldg(hw + n * r + o) * relu_if(__ldg(acts + n * d + i), relu);
  }
};
struct RecordV {  // materialised per-sample values: v(n, j) = g[n, j]
  const float* g;
  int64_t numel;
  __device__ __forceinline__ float operator()(int64_t n, int64_t j) const { return __ldg(g + n * numel + j); }
};

__global__ void __launch_bounds__(32 * kColWarps) wsum_outer_kernel(OuterV v, const float* scale, int64_t b,
                                                                    float* out, int accumulate) {
  pdl_wait();
  colsum_body(v, ScaleC{scale}, b, v.d * v.r, (int64_t)blockIdx.x * 32, out, accumulate);
}

// all small per-sample records (the biases) of a model in one launch: blockIdx.y = item
__global__ void __launch_bounds__(32 * kColWarps) wsum_multi_kernel(WsumItems items, const float* scale,
                                                                    int64_t b, int accumulate) {
  pdl_wait();
  const WsumItem& it = items.item[blockIdx.y];
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  if (j0 >= it.numel) return;
  colsum_body(RecordV{it.g, it.numel}, ScaleC{scale}, b, it.numel, j0, it.out, accumulate);
}

void launch_wsum_multi(dpg_ctx* ctx, const WsumItems& items, const float* scale, int64_t b,
                       int accumulate) {
  if (items.count == 0) return;
  int64_t maxn = 0;
  for (int i = 0; i < items.count; ++i) maxn = items.item[i].numel > maxn ? items.item[i].numel : maxn;
  dim3 grid((unsigned)((maxn + 31) / 32), (unsigned)items.count);
  ::dpg::launch_pdl(wsum_multi_kernel, grid, 32 * kColWarps, 0, ctx->stream, items, scale, b, accumulate);
  DPG_LAUNCH_CHECK(ctx);
}

// Linear weight, mid > 1: split-K GEMM over (n, t).
size_t clipped_sum_ws_linear(int64_t b, int64_t mid, int64_t d, int64_t r) {
  if (mid == 1) return 0;
  int splits = tc::csum_linear_splits(b, mid, d, r);
  if (tg::lin_shape_ok(b, mid, d, r)) splits = std::max(splits, tg::lin_csum_splits(b, mid, d, r));
  return sizeof(float) * (size_t)splits * (size_t)(r * d);
}

void launch_clipped_sum_linear(dpg_ctx* ctx, const float* acts, int acts_relu, const float* hw,
                               const float* scale, int64_t b, int64_t mid, int64_t d, int64_t r,
                               float* sw, float* sb, int accumulate, void* ws) {
  (void)sb;  // the bias sum is formed from the per-sample bias record (launch_weighted_sum_...)
  if (mid == 1) {
    if (d * r >= (int64_t(1) << 31)) raise(DPG_ERR_DIMENSION, "linear clipped sum: d * r too large");
    OuterV v{acts, hw, d, r, acts_relu};
    ::dpg::launch_pdl(wsum_outer_kernel, (unsigned)((r * d + 31) / 32), 32 * kColWarps, 0, ctx->stream, v, scale, b, sw, accumulate);
    DPG_LAUNCH_CHECK(ctx);
    return;
  }
  if (tg::lin_ok(acts, hw, ws, b, mid, d, r)) {  // TMA-fed core, partials [split][o][i] as below
    const int splits = tg::lin_csum_splits(b, mid, d, r);
    tg::lin_csum(ctx, acts, acts_relu, hw, scale, b, mid, d, r, static_cast<float*>(ws), splits);
    launch_splitk_reduce(ctx, static_cast<float*>(ws), splits, r * d, sw, accumulate);
    return;
  }
  const int splits = tc::csum_linear_splits(b, mid, d, r);
  tc::linear_csum(ctx, acts, acts_relu, hw, scale, b, mid, d, r, static_cast<float*>(ws), splits);
  launch_splitk_reduce(ctx, static_cast<float*>(ws), splits, r * d, sw, accumulate);
}

// ------------------------------------------------------------------------------------------
// Conv weight: S[oc, k] = sum_{n, p} (scale_n * B[n, oc, p]) * X~[n, k, p] — the conv weight
// gradient of the clip-scaled highway; split-K over samples.
// ------------------------------------------------------------------------------------------
size_t clipped_sum_ws_conv2d(const ConvGeom& g, bool nhwc_in) {
  if (nhwc_in) return sizeof(float) * (size_t)tg::csum_nhwc_splits(g) * (size_t)(g.oc * g.K());
  if (tk::supported(g)) return sizeof(float) * (size_t)tk::csum_splits(g) * (size_t)(g.oc * g.K());
  return sizeof(float) * (size_t)tc::csum_conv_splits(g) * (size_t)(g.oc * g.K());
}

void launch_clipped_sum_conv2d(dpg_ctx* ctx, const float* x, int x_relu, const float* hw,
                               const float* scale, const ConvGeom& g, float* sw, float* sb,
                               int accumulate, void* ws, bool hw_nhwc, const float* xh) {
  (void)sb;  // the bias clipped sum is a weighted sum of the bias records (launch_wsum_multi)
  const int64_t nw = g.oc * g.K();
  if (xh) {  // the layer input's NHWC copy exists: the TMA-fed core (tg_conv.cu ConvCsumT)
    if (hw_nhwc || !tg::csum_nhwc_ok(g)) raise(DPG_ERR_INTERNAL, "NHWC clipped sum: unsupported geometry");
    const int splits = tg::csum_nhwc_splits(g);
    tg::conv_csum_nhwc(ctx, xh, hw, scale, g, static_cast<float*>(ws), splits);
    if (launch_splitk_reduce4(ctx, static_cast<float*>(ws), splits, nw, sw, accumulate,
                              TapMajorOut{(int)g.ic, (int)(g.kh * g.kw), g.K()}))
      return;
    ::dpg::launch_pdl(splitk_reduce_tap_kernel, (unsigned)((nw + 31) / 32), 32 * kColWarps, 0, ctx->stream,
                      PartV{static_cast<float*>(ws), nw}, splits, nw, sw, accumulate,
                      TapMajorOut{(int)g.ic, (int)(g.kh * g.kw), g.K()});
    DPG_LAUNCH_CHECK(ctx);
    return;
  }
  if (hw_nhwc && !tk::supported(g)) raise(DPG_ERR_INTERNAL, "channels-last highway needs the thin-K path");
  if (tk::supported(g)) {
    const int splits = tk::csum_splits(g);
    tk::csum(ctx, x, x_relu, hw, scale, g, static_cast<float*>(ws), splits, hw_nhwc);
    launch_splitk_reduce(ctx, static_cast<float*>(ws), splits, nw, sw, accumulate);
    return;
  }
  const int splits = tc::csum_conv_splits(g);
  tc::conv_csum(ctx, x, x_relu, hw, scale, g, static_cast<float*>(ws), splits);
  launch_splitk_reduce(ctx, static_cast<float*>(ws), splits, nw, sw, accumulate);
}

// ------------------------------------------------------------------------------------------
// Embedding: summed[v, :] = sum_n scale_n * G_n[v, :], G_n[v] = sum over sample n's duplicates
// of v in ascending s — exactly the reference's order (grad_sample.hpp:74-80 then
// optimizer.hpp:107-110), so bit-exact. Stage 1 builds start[n][c] = first sorted position of
// sample n in vocab chunk c; stage 2 gives each CTA one chunk of kCsRows rows, warps own rows,
// samples are visited in ascending order.
// ------------------------------------------------------------------------------------------
constexpr int kCsRows = 32;

__global__ void embed_chunk_starts_kernel(const int32_t* __restrict__ sorted_v, int64_t t,
                                          int nchunks, int32_t* __restrict__ starts) {
  pdl_wait();
  const int64_t n = blockIdx.x;
  const int32_t* sv = sorted_v + n * t;
  for (int c = threadIdx.x; c <= nchunks; c += blockDim.x) {
    const int32_t v = (int32_t)((int64_t)c * kCsRows);
    int lo = 0, hi = (int)t;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sv[mid] < v) lo = mid + 1; else hi = mid;
    }
    starts[n * (nchunks + 1) + c] = lo;
  }
}

// Stage 2: the chunk's work list is staged in shared memory first — per-sample entry counts
// (from the stage-1 starts), their exclusive prefix sum, and the (row, position) pairs of every
// sample's tokens that fall in the chunk, in sample order — so the ordered accumulation loop only
// touches global memory for the highway rows (no dependent index loads per sample). Chunks with
// more entries than fit fall back to reading the indices from global memory.
constexpr int kCsMaxEntries = 4096;

__global__ void __launch_bounds__(256, 3) clipped_sum_embedding_kernel(
    const int32_t* __restrict__ sorted_v, const int32_t* __restrict__ sorted_s,
    const int32_t* __restrict__ starts, const float* __restrict__ hw,
    const float* __restrict__ scale, int64_t b, int64_t t, int64_t vocab, int64_t dim,
    int nchunks, float* __restrict__ summed, int accumulate) {
  pdl_wait();
  extern __shared__ float acc[];  // [kCsRows][dim], then the work list
  int* cnt = reinterpret_cast<int*>(acc + kCsRows * dim);  // [b + 1] exclusive prefix of entries
  int* ev = cnt + (b + 1);                                 // [kCsMaxEntries] row - v0
  int* es = ev + kCsMaxEntries;                            // [kCsMaxEntries] position s
  int* en = es + kCsMaxEntries;                            // [kCsMaxEntries] sample n
  __shared__ int total_sh;
  const int c = blockIdx.x;
  const int64_t v0 = (int64_t)c * kCsRows;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int64_t i = tid; i < kCsRows * dim; i += 256) acc[i] = 0.f;
  // per-sample entry counts, then an exclusive scan: each thread sums a contiguous block of
  // samples, the 256 block sums are scanned by warp shuffles, then each block is re-walked
  __shared__ int wsum[8];
  const int64_t per = (b + 255) / 256, nb0 = tid * per, nb1 = nb0 + per < b ? nb0 + per : b;
  int mine = 0;
  for (int64_t n = nb0; n < nb1; ++n) {
    const int m = starts[n * (nchunks + 1) + c + 1] - starts[n * (nchunks + 1) + c];
    cnt[n + 1] = m;
    mine += m;
  }
  int incl = mine;  // inclusive warp scan of the per-thread sums
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  int run = base + incl - mine;  // exclusive prefix of this thread's block
  if (tid == 0) cnt[0] = 0;
  for (int64_t n = nb0; n < nb1; ++n) {
    run += cnt[n + 1];
    cnt[n + 1] = run;
  }
  if (tid == 255) total_sh = run;
  __syncthreads();
  const int total = total_sh;
  const bool staged = total <= kCsMaxEntries;
  if (staged) {
    for (int64_t n = tid; n < b; n += 256) {  // a thread per sample: copy its (few) entries
      const int j0 = starts[n * (nchunks + 1) + c], e0 = cnt[n], m = cnt[n + 1] - e0;
      for (int q = 0; q < m; ++q) {
        ev[e0 + q] = sorted_v[n * t + j0 + q] - (int)v0;
        es[e0 + q] = sorted_s[n * t + j0 + q];
        en[e0 + q] = (int)n;
      }
    }
  }
  __syncthreads();
  if (staged && kCsRows * 8 == 256 && (dim % 32) == 0 && dim <= 128) {
    // thread (row r = tid / 8, slice = tid % 8 of dim / 8 columns): walk the chunk's entries in
    // sample order and accumulate the ones of row r — each thread only waits on its own row's
    // ~b t / vocab highway loads, and the 256 threads' loads are independent
    const int r = tid >> 3, w8 = (int)(dim >> 3), d0 = (tid & 7) * w8;
    float a[16], gsum[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a[k] = 0.f;
      gsum[k] = 0.f;
    }
    int cur_n = -1;
    // matching entries are gathered in batches of kB and their highway loads issued together,
    // then accumulated in order (runs of one sample summed first, then scaled in)
    constexpr int kB = 2;
    int bn[kB], bs[kB];
    int nb = 0;
    auto flush = [&]() {
      float4 h[kB][4];
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (q < nb) {
          const float* src = hw + ((int64_t)bn[q] * t + bs[q]) * dim + d0;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (4 * k < w8) h[q][k] = __ldg(reinterpret_cast<const float4*>(src + 4 * k));
        }
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (q < nb) {
          if (bn[q] != cur_n) {
            if (cur_n >= 0) {
              const float w = __ldg(scale + cur_n);
#pragma unroll
              for (int k = 0; k < 16; ++k)
                if (k < w8) a[k] = __fadd_rn(a[k], __fmul_rn(w, gsum[k]));
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) gsum[k] = 0.f;
            cur_n = bn[q];
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (4 * k < w8) {
              gsum[4 * k] = __fadd_rn(gsum[4 * k], h[q][k].x);
              gsum[4 * k + 1] = __fadd_rn(gsum[4 * k + 1], h[q][k].y);
              gsum[4 * k + 2] = __fadd_rn(gsum[4 * k + 2], h[q][k].z);
              gsum[4 * k + 3] = __fadd_rn(gsum[4 * k + 3], h[q][k].w);
            }
        }
      nb = 0;
    };
    for (int e = 0; e < total; ++e) {
      if (ev[e] != r) continue;
      bn[nb] = en[e];
      bs[nb] = es[e];
      if (++nb == kB) flush();
    }
    flush();
    if (cur_n >= 0) {
      const float w = __ldg(scale + cur_n);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < w8) a[k] = __fadd_rn(a[k], __fmul_rn(w, gsum[k]));
    }
    if (v0 + r < vocab) {
      float* o = summed + (v0 + r) * dim + d0;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < w8) o[k] = accumulate ? __fadd_rn(o[k], a[k]) : a[k];
    }
    return;
  }
  for (int64_t n = 0; n < b; ++n) {
    const int e0 = cnt[n], e1 = cnt[n + 1];
    if (e0 == e1) continue;
    const float w = __ldg(scale + n);
    const int j0 = staged ? 0 : starts[n * (nchunks + 1) + c];
    const int32_t* sv = sorted_v + n * t;
    const int32_t* ss = sorted_s + n * t;
    const float* hwn = hw + n * t * dim;
    for (int e = e0; e < e1;) {
      const int r = staged ? ev[e] : sv[j0 + e - e0] - (int)v0;
      int f = e + 1;
      while (f < e1 && (staged ? ev[f] : sv[j0 + f - e0] - (int)v0) == r) ++f;
      if ((r & 7) == warp) {
        float* arow = acc + r * dim;
        for (int64_t d0 = lane; d0 < dim; d0 += 32) {
          float g = 0.f;
          for (int q = e; q < f; ++q) {
            const int sp = staged ? es[q] : ss[j0 + q - e0];
            g = __fadd_rn(g, __ldg(hwn + (int64_t)sp * dim + d0));
          }
          arow[d0] = __fadd_rn(arow[d0], __fmul_rn(w, g));
        }
      }
      e = f;
    }
  }
  __syncthreads();
  for (int64_t i = tid; i < kCsRows * dim; i += 256) {
    const int64_t v = v0 + i / dim;
    if (v >= vocab) break;
    float* o = summed + v0 * dim + i;
    *o = accumulate ? __fadd_rn(*o, acc[i]) : acc[i];
  }
}

size_t clipped_sum_ws_embedding(int64_t b, int64_t vocab) {
  const int64_t nchunks = (vocab + kCsRows - 1) / kCsRows;
  return sizeof(int32_t) * (size_t)(b * (nchunks + 1));
}

void launch_clipped_sum_embedding(dpg_ctx* ctx, const int32_t* sorted_v, const int32_t* sorted_s,
                                  const float* hw, const float* scale, int64_t b, int64_t t,
                                  int64_t vocab, int64_t dim, float* summed, int accumulate,
                                  void* ws) {
  const int nchunks = (int)((vocab + kCsRows - 1) / kCsRows);
  int32_t* starts = static_cast<int32_t*>(ws);
  if (b > 0) {
    ::dpg::launch_pdl(embed_chunk_starts_kernel, (unsigned)b, 256, 0, ctx->stream, sorted_v, t, nchunks, starts);
    DPG_LAUNCH_CHECK(ctx);
  }
  const size_t smem = sizeof(float) * kCsRows * (size_t)dim + sizeof(int) * ((size_t)b + 1 + 3 * kCsMaxEntries);
  if (smem > 200 * 1024) raise(DPG_ERR_DIMENSION, "clipped_sum_embedding: batch or embedding_dim too large for one chunk");
  if (smem > 48 * 1024)
    ensure_smem_attr(reinterpret_cast<const void*>(clipped_sum_embedding_kernel), (int)smem);
  ::dpg::launch_pdl(clipped_sum_embedding_kernel, (unsigned)nchunks, 256, smem, ctx->stream, 
      sorted_v, sorted_s, starts, hw, scale, b, t, vocab, dim, nchunks, summed, accumulate);
  DPG_LAUNCH_CHECK(ctx);
}

// ------------------------------------------------------------------------------------------
// Materialised record (reference pass 1 and pass 2 over stored per-sample gradients).
// ------------------------------------------------------------------------------------------
constexpr int64_t kSqChunk = 16384;

__global__ void __launch_bounds__(256) sq_materialised_kernel(const float* __restrict__ g,
                                                              int64_t b, int64_t numel,
                                                              double* __restrict__ sq_part) {
  pdl_wait();
  const int64_t n = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * kSqChunk;
  const int64_t c1 = c0 + kSqChunk < numel ? c0 + kSqChunk : numel;
  const float* row = g + n * numel;
  double sq = 0.0;
  for (int64_t j = c0 + threadIdx.x; j < c1; j += 256) {
    const double v = (double)__ldg(row + j);
    sq += v * v;
  }
  __shared__ double red[8];
  const double t = block_sum<256>(sq, red);
  if (threadIdx.x == 0) sq_part[(int64_t)blockIdx.x * b + n] = t;
}

int sq_rows_materialised(int64_t numel) { return (int)((numel + kSqChunk - 1) / kSqChunk); }

void launch_sq_materialised(dpg_ctx* ctx, const float* g, int64_t b, int64_t numel,
                            double* sq_part) {
  if (b == 0) return;
  dim3 grid((unsigned)sq_rows_materialised(numel), (unsigned)b);
  ::dpg::launch_pdl(sq_materialised_kernel, grid, 256, 0, ctx->stream, g, b, numel, sq_part);
  DPG_LAUNCH_CHECK(ctx);
}

// summed[j] = [summed[j] +] sum_n (float)scale_n * g[n, j], n ascending (optimizer.hpp:106-111)
__global__ void weighted_sum_kernel(const float* __restrict__ g, const float* __restrict__ scale,
                                    int64_t b, int64_t numel, float* __restrict__ summed,
                                    int accumulate) {
  pdl_wait();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= numel) return;
  // the reference's sequential order, with 16 samples' loads in flight per round (a streaming
  // read of the record instead of one dependent HBM latency per sample)
  float acc = 0.f;
  int64_t n = 0;
  for (; n + 16 <= b; n += 16) {
    float v[16], s[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      v[u] = __ldg(g + (n + u) * numel + j);
      s[u] = __ldg(scale + n + u);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, __fmul_rn(s[u], v[u]));
  }
  for (; n < b; ++n) acc = __fadd_rn(acc, __fmul_rn(__ldg(scale + n), __ldg(g + n * numel + j)));
  summed[j] = accumulate ? __fadd_rn(summed[j], acc) : acc;
}

// Narrow parameters (a few thousand columns): the record is staged through shared memory in
// 64-sample chunks loaded by the whole CTA (every load in flight at once), then each thread
// sums its column over the chunk in sample order — same order and roundings as above.
constexpr int kWsCols = 32, kWsChunk = 128;
__global__ void __launch_bounds__(256) weighted_sum_narrow_kernel(const float* __restrict__ g,
                                                                  const float* __restrict__ scale, int64_t b,
                                                                  int64_t numel, float* __restrict__ summed,
                                                                  int accumulate) {
  pdl_wait();
  __shared__ float tile[kWsChunk][kWsCols + 1];
  __shared__ float sc[kWsChunk];
  const int64_t j0 = (int64_t)blockIdx.x * kWsCols;
  const int tid = threadIdx.x;
  float acc = 0.f;
  for (int64_t n0 = 0; n0 < b; n0 += kWsChunk) {
    const int nn = (int)(b - n0 < kWsChunk ? b - n0 : kWsChunk);
    {  // lane = column, warp w = samples w, w + 8, ...: 16 coalesced loads in flight per thread
      const int c = tid & 31, q0 = tid >> 5;
      float v[kWsChunk / 8];
#pragma unroll
      for (int u = 0; u < kWsChunk / 8; ++u) {
        const int q = q0 + 8 * u;
        v[u] = (q < nn && j0 + c < numel) ? __ldg(g + (n0 + q) * numel + j0 + c) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kWsChunk / 8; ++u) tile[q0 + 8 * u][c] = v[u];
    }
    if (tid < kWsChunk) sc[tid] = tid < nn ? __ldg(scale + n0 + tid) : 0.f;
    __syncthreads();
    if (tid < kWsCols)
      for (int q = 0; q < nn; ++q) acc = __fadd_rn(acc, __fmul_rn(sc[q], tile[q][tid]));
    __syncthreads();
  }
  const int64_t j = j0 + tid;
  if (tid < kWsCols && j < numel) summed[j] = accumulate ? __fadd_rn(summed[j], acc) : acc;
}

void launch_weighted_sum_materialised(dpg_ctx* ctx, const float* g, const float* scale, int64_t b,
                                      int64_t numel, float* summed, int accumulate) {
  if (numel == 0) return;
  if (numel <= 8192) {
    ::dpg::launch_pdl(weighted_sum_narrow_kernel, (unsigned)((numel + kWsCols - 1) / kWsCols), 256, 0, ctx->stream,
                      g, scale, b, numel, summed, accumulate);
    DPG_LAUNCH_CHECK(ctx);
    return;
  }
  ::dpg::launch_pdl(weighted_sum_kernel, (unsigned)((numel + 255) / 256), 256, 0, ctx->stream, g, scale, b, numel, summed, accumulate);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace dpg
