// rows_conv.cu — per-sample conv gradients for layers with few positions per sample (P <= 16).
//
//   G[n][oc][kcol] = sum_p B[n, oc, p] X~[n, kcol, p]     (per_sample_rule_conv2d,
//                    grad_sample.hpp:135-150) + the fused ||G_n||^2 partial
//   gb[n][oc]      = (float) sum_p (double) B[n, oc, p]   (bias rule, sum_middle order,
//                    tensor.hpp:197-205) + its squared norm
//
// With P <= 16 every output costs at most 16 MACs, so the layer is bound by the HBM write of G
// (the largest stream of the whole step: CIFAR conv4 alone is 151 MB at b = 512). The kernel is
// built around that store stream: one CTA owns one sample and a contiguous half (or all) of its
// output channels; im2col of the sample (P x Kc, ReLU applied) and the highway rows of its channels
// are staged once in shared memory (the highway tile transposed, [p][oc]); then each warp produces
// 4 output rows at a time — lanes walk the rows in 16-byte chunks, every chunk is P pairs of
// 128-bit shared reads (im2col, and the 4 rows' highway values as a broadcast), 16 P FMAs and four
// 128-bit streaming stores, so consecutive lanes write consecutive 16 B of G (512 B per store).
#include <cstdlib>

#include "conv_common.cuh"

namespace dpg {
namespace rs {

constexpr int kThreads = 256;
constexpr int kMaxP = 16;

struct Params {
  const float* x;
  int relu;
  const float* hw;
  float* gw;         // [b, oc, Kc] (nullptr: norms only)
  double* sq_part;   // [osplit, b]
  float* gb;         // [b, oc] (nullptr: no bias record)
  double* sq_b;      // [osplit, b] (nullptr: no bias rule)
  int64_t b;
  int ic, h, w, oc, kh, kw, stride, pad, ow, P, Kc, Kc4, osplit, opart;
};

template <int PT>
__global__ void __launch_bounds__(kThreads, 4) gs_rows_kernel(const Params p) {
  
  extern __shared__ __align__(16) float sm[];
  float* xt = sm;                                          // [PT][Kc4], rows >= P are zero
  const int ostr = (p.opart + 3) & ~3;                     // row stride of the transposed tile
  float* hs = xt + PT * p.Kc4;                             // [PT][ostr] = B[n, o, q] transposed
  int* kt = reinterpret_cast<int*>(hs + PT * ostr);        // [Kc4] packed (c, ki, kj) or -1
  __shared__ double red[2][kThreads / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = blockIdx.y;
  const int part = blockIdx.x;
  const int o_begin = part * p.opart;
  const int o_end = min(p.oc, o_begin + p.opart);
  const int nrow = o_end - o_begin;
  const int hwsz = p.h * p.w;

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
  pdl_wait();  // the tap table above is geometry only
  // highway rows of this part: contiguous [nrow][P] in B[n]
  const float* hrow = p.hw + ((int64_t)n * p.oc + o_begin) * p.P;
  for (int i = tid; i < ostr * PT; i += kThreads) {
    const int o = i / PT, q = i - o * PT;  // coalesced global reads, transposed shared stores
    hs[q * ostr + o] = (q < p.P && o < nrow) ? __ldg(hrow + o * p.P + q) : 0.f;
  }
  __syncthreads();
  // im2col of sample n: xt[q][k] = relu(x[n, c, oy s + ki - pad, ox s + kj - pad])
  const float* xn = p.x + n * p.ic * hwsz;
  int by[PT], bx[PT];  // window origin of each position
#pragma unroll
  for (int q = 0; q < PT; ++q) {
    const int oy = q / p.ow, ox = q - oy * p.ow;
    by[q] = oy * p.stride - p.pad;
    bx[q] = ox * p.stride - p.pad;
  }
  for (int k = tid; k < p.Kc4; k += kThreads) {
    const int e = kt[k];
    const int coff = (e >> 10) * hwsz, ki = (e >> 5) & 31, kj = e & 31;
    float v[PT];
#pragma unroll
    for (int q = 0; q < PT; ++q) {  // all PT loads in flight, then ReLU and store
      const int iy = by[q] + ki, ix = bx[q] + kj;
      const bool ok = e >= 0 && q < p.P && (unsigned)iy < (unsigned)p.h && (unsigned)ix < (unsigned)p.w;
      v[q] = ldg_or_zero(xn + (coff + iy * p.w + ix), ok);
    }
#pragma unroll
    for (int q = 0; q < PT; ++q) xt[q * p.Kc4 + k] = relu_if(v[q], p.relu);
  }
  __syncthreads();

  double sq = 0.0, sqb = 0.0;
  const int nq = p.Kc4 >> 2;
  const bool vec = (p.Kc & 3) == 0;
  // 4 rows per warp pass: per position, one 128-bit im2col read and one 128-bit (broadcast) read
  // of the 4 rows' highway values feed 16 FMAs; few registers, so several CTAs share an SM and
  // one's staging overlaps another's stores
  constexpr int R = 4;
  for (int r0 = R * warp; r0 < nrow; r0 += R * (kThreads / 32)) {
    if (p.sq_b && lane < R && r0 + lane < nrow) {
      // bias rule for row r0 + lane: sequential fp64 sum over the P positions
      const float* hb = hs + r0 + lane;
      double a = 0.0;
      for (int q = 0; q < p.P; ++q) a += (double)hb[q * ostr];
      const float v = (float)a;
      if (p.gb) p.gb[n * p.oc + o_begin + r0 + lane] = v;
      sqb += (double)v * v;
    }
    float* g0 = p.gw ? p.gw + (n * p.oc + o_begin + r0) * (int64_t)p.Kc : nullptr;
    for (int j = lane; j < nq; j += 32) {
      float4 acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < PT; ++q) {
        const float4 xv = *reinterpret_cast<const float4*>(xt + q * p.Kc4 + 4 * j);
        const float4 b4 = *reinterpret_cast<const float4*>(hs + q * ostr + r0);
        const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r].x = fmaf(bv[r], xv.x, acc[r].x); acc[r].y = fmaf(bv[r], xv.y, acc[r].y);
          acc[r].z = fmaf(bv[r], xv.z, acc[r].z); acc[r].w = fmaf(bv[r], xv.w, acc[r].w);
        }
      }
      const int k0 = 4 * j;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r0 + r >= nrow) break;
        const float4 a = acc[r];
        if (vec) {
          if (g0) st_stream4(g0 + (int64_t)r * p.Kc + k0, a);
          sq += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
        } else {
          const float v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (k0 + e >= p.Kc) break;
            if (g0) st_stream(g0 + (int64_t)r * p.Kc + k0 + e, v[e]);
            sq += (double)v[e] * v[e];
          }
        }
      }
    }
  }
  // deterministic block sums (fixed tree)
  sq = warp_sum(sq);
  sqb = warp_sum(sqb);
  if (lane == 0) {
    red[0][warp] = sq;
    red[1][warp] = sqb;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0, tb = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) {
      t += red[0][i];
      tb += red[1][i];
    }
    if (p.sq_part) p.sq_part[(int64_t)part * p.b + n] = t;
    if (p.sq_b) p.sq_b[(int64_t)part * p.b + n] = tb;
  }
}

static int pick_pt(int P) { return P <= 4 ? 4 : (P <= 8 ? 8 : 16); }

static Params make_params(const float* x, int relu, const float* hw, const ConvGeom& g) {
  Params p{};
  p.x = x; p.relu = relu; p.hw = hw;
  p.b = g.b;
  p.ic = (int)g.ic; p.h = (int)g.h; p.w = (int)g.w; p.oc = (int)g.oc;
  p.kh = (int)g.kh; p.kw = (int)g.kw; p.stride = (int)g.stride; p.pad = (int)g.pad;
  p.ow = (int)g.ow; p.P = (int)g.P(); p.Kc = (int)g.K();
  p.Kc4 = (p.Kc + 3) & ~3;
  // two channel halves per sample for wide layers with few positions (cheap im2col): twice the
  // CTAs (shorter tail), im2col built twice
  p.osplit = (g.oc >= 64 && g.P() <= 8) ? 2 : 1;
  p.opart = (int)((g.oc + p.osplit - 1) / p.osplit);
  return p;
}

static size_t smem_bytes(const Params& p) {
  const int PT = pick_pt(p.P);
  return sizeof(float) * ((size_t)PT * p.Kc4 + (size_t)PT * ((p.opart + 3) & ~3)) + sizeof(int) * (size_t)p.Kc4;
}

bool supported(const ConvGeom& g) {
  if (g.P() > kMaxP || g.kh >= 32 || g.kw >= 32 || g.ic >= (1 << 21)) return false;
  return smem_bytes(make_params(nullptr, 0, nullptr, g)) <= 160 * 1024;
}

int gs_rows(const ConvGeom& g) { return make_params(nullptr, 0, nullptr, g).osplit; }

void gs(dpg_ctx* ctx, const float* x, int relu, const float* hw, const ConvGeom& g, float* gw,
        double* sq_part, float* gb, double* sq_b) {
  Params p = make_params(x, relu, hw, g);
  p.gw = gw;
  p.sq_part = sq_part;
  p.gb = gb;
  p.sq_b = (gb || sq_b) ? sq_b : nullptr;
  if (gb && !sq_b) raise(DPG_ERR_INTERNAL, "rs::gs: bias record without its norm rows");
  const size_t smem = smem_bytes(p);
  dim3 grid((unsigned)p.osplit, (unsigned)g.b);
  auto go = [&](auto kern) {
    ensure_smem_attr(reinterpret_cast<const void*>(kern), (int)smem);
    ::dpg::launch_pdl(kern, grid, kThreads, smem, ctx->stream, p);
  };
  switch (pick_pt(p.P)) {
    case 4: go(gs_rows_kernel<4>); break;
    case 8: go(gs_rows_kernel<8>); break;
    default: go(gs_rows_kernel<16>); break;
  }
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace rs
}  // namespace dpg
