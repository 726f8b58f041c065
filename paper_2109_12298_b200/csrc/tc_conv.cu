// tc_conv.cu — the dense contractions of the step on tcgen05 (3xTF32, tc_gemm.cuh):
//
//   conv forward      Y[(n,p), oc]    = sum_kcol X~[n, kcol, p] W[oc, kcol]   (+ bias)
//   conv dgrad        dX[(n,pix), c]  = sum_(oc,tap) dY[n, oc, o(pix,tap)] W[oc, c, tap]
//                     per stride-parity class of input pixels (no wasted taps), ReLU mask fused
//   per-sample conv   G[n][oc][kcol]  = sum_p X~[n, kcol, p] B[n, oc, p]   + fused ||G_n||^2
//   clipped conv sum  S[oc][kcol]     = sum_(n,p) X~[n, kcol, p] (s_n B[n, oc, p])  (split over n)
//   per-sample linear G[n][o][i]      = sum_t A[n, t, i] B[n, t, o]           (mid > 1)
//   clipped linear    S[o][i]         = sum_(n,t) A[n, t, i] (s_n B[n, t, o])  (split over n)
//
// The GEMM row dimension (UMMA M = 128 TMEM lanes) is always the dimension that is contiguous in
// the output, so each warp's epilogue stores are coalesced. The implicit-im2col index maps are
// precomputed once per CTA into shared-memory tables (k -> plane offset / tap, p -> (oy s, ox s),
// row -> base offset), so each gathered element costs one broadcast table read, two bound checks
// and one load.
#include <cstdlib>

#include "conv_common.cuh"
#include "tc_gemm.cuh"

namespace dpg {
namespace tc {

struct Geo {
  int ic, h, w, oc, kh, kw, stride, pad, oh, ow;
  int64_t P, Kc;
  FastDiv fP, fow;
};

inline Geo make_geo(const ConvGeom& g) {
  Geo r;
  r.ic = (int)g.ic; r.h = (int)g.h; r.w = (int)g.w; r.oc = (int)g.oc;
  r.kh = (int)g.kh; r.kw = (int)g.kw; r.stride = (int)g.stride; r.pad = (int)g.pad;
  r.oh = (int)g.oh; r.ow = (int)g.ow;
  r.P = g.P();
  r.Kc = g.K();
  r.fP = FastDiv((uint32_t)g.P());
  r.fow = FastDiv((uint32_t)g.ow);
  return r;
}

// kcol -> offset of (c, ki, kj) relative to a window origin, and the tap (ki, kj)
struct KEnt {  // (read back as one int2: {off, ki | kj << 16})
  int off;
  short ki, kj;
};
// position p -> window origin (oy s - pad, ox s - pad)
struct PEnt {
  short y, x;
};

constexpr int kBad = -(1 << 14);

__device__ __forceinline__ float4 relu4(float4 v, int relu) {
  return make_float4(relu_if(v.x, relu), relu_if(v.y, relu), relu_if(v.z, relu), relu_if(v.w, relu));
}
#define DPG_NO_FIX(NAME) \
  __device__ float4 NAME(int, int64_t, int, int64_t, const uint8_t*, float4 v) const { return v; }  // sentinel coordinate: (unsigned)(kBad + small) >= h, w

// k-table for kcol 0 .. kpad (entries >= K are sentinels that fail every bound check)
__device__ __forceinline__ void build_ktab(const Geo& g, KEnt* t, int tid, int K, int kpad) {
  for (int k = tid; k < kpad; k += kThreads) {
    if (k < K) {
      const int khw = g.kh * g.kw;
      const int c = k / khw, r = k - c * khw;
      const int ki = r / g.kw, kj = r - ki * g.kw;
      t[k] = KEnt{(c * g.h + ki) * g.w + kj, (short)ki, (short)kj};
    } else {
      t[k] = KEnt{0, (short)kBad, (short)kBad};
    }
  }
}
__device__ __forceinline__ void build_ptab(const Geo& g, PEnt* t, int tid) {
  for (int p = tid; p < ((g.P + 3) & ~3); p += kThreads) {
    const int oy = p / g.ow, ox = p - oy * g.ow;
    // the padding up to a multiple of 4 holds sentinels, so a quad is one 16-byte load
    t[p] = p < g.P ? PEnt{(short)(oy * g.stride - g.pad), (short)(ox * g.stride - g.pad)}
                   : PEnt{(short)kBad, (short)kBad};
  }
}
__device__ __forceinline__ void ptab_quad(const PEnt* pt, int p, PEnt (&t)[4]) {
  const int4 q = *reinterpret_cast<const int4*>(pt + p);
  t[0] = *reinterpret_cast<const PEnt*>(&q.x);
  t[1] = *reinterpret_cast<const PEnt*>(&q.y);
  t[2] = *reinterpret_cast<const PEnt*>(&q.z);
  t[3] = *reinterpret_cast<const PEnt*>(&q.w);
}

// The gathers use 32-bit element offsets: every tensor a contraction reads must have < 2^31
// elements (2^31 floats = 8 GiB; the per-sample gradient record is written with 64-bit offsets).
static void check_i32(const ConvGeom& cg) {
  const int64_t lim = int64_t(1) << 31;
  if (cg.b * cg.ic * cg.h * cg.w >= lim || cg.b * cg.oc * cg.P() >= lim || cg.oc * cg.K() >= lim)
    raise(DPG_ERR_DIMENSION, "conv2d: a tensor of this batch exceeds 2^31 elements");
}
static void check_i32_linear(int64_t b, int64_t mid, int64_t d, int64_t r) {
  const int64_t lim = int64_t(1) << 31;
  if (b * mid * d >= lim || b * mid * r >= lim || d * r >= lim)
    raise(DPG_ERR_DIMENSION, "linear: a tensor of this batch exceeds 2^31 elements");
}

// ------------------------------------------------------------------------------ forward
struct ConvFwd : TileRows {
  static constexpr bool kCtaReduce = false;
  Geo g;
  const float* x;
  int relu;
  const float* wt;
  const float* bias;
  float* y;
  float* yh;     // NHWC [b][P][oc] of relu_if(y, relu_out) for a TMA-fed consumer (nullable)
  int relu_out;
  float* part;  // split-K partials [ksplit][oc][M] (ksplit > 1)
  int64_t M, N, K;
  int ksplit, scratch;
  struct Row {
    const float* xr;  // x + n*ic*h*w + iy0*w + ix0
    int iy0, ix0;     // window origin; kBad for rows beyond M (every bound check fails)
  };
  __device__ int64_t mdim(int) const { return M; }
  __device__ int64_t kdim(int) const { return K; }
  __device__ int ktab_bytes() const { return (int)(8 * ((K + BK - 1) / BK) * BK); }
  __device__ void setup(int, int64_t m0, int64_t, uint8_t* s, int tid) const {
    KEnt* kt = reinterpret_cast<KEnt*>(s);
    Row* rows = reinterpret_cast<Row*>(s + ktab_bytes());
    build_ktab(g, kt, tid, (int)K, (int)((K + BK - 1) / BK) * BK);
    if (tid < BM) {
      Row r{x, kBad, kBad};
      if (m0 + tid < M) {
        uint32_t n, p, oy, ox;
        g.fP.divmod((uint32_t)(m0 + tid), n, p);
        g.fow.divmod(p, oy, ox);
        const int iy0 = (int)oy * g.stride - g.pad, ix0 = (int)ox * g.stride - g.pad;
        r = Row{x + (int64_t)n * g.ic * g.h * g.w + (int64_t)iy0 * g.w + ix0, iy0, ix0};
      }
      rows[tid] = r;
    }
  }
  static constexpr bool kAQuadMajor = false;  // rows = output positions: lanes walk ox
  static constexpr bool kBQuadMajor = true;   // W rows contiguous in kcol
  __device__ float4 a_quad(int, int64_t, int row, int64_t k, const uint8_t* s) const {
    const KEnt* kt = reinterpret_cast<const KEnt*>(s) + (int)k;
    const Row r = reinterpret_cast<const Row*>(s + ktab_bytes())[row];
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int2 t = *reinterpret_cast<const int2*>(kt + e);  // one 64-bit read: {off, ki | kj << 16}
      const int ki = (int)(short)(t.y & 0xffff), kj = t.y >> 16;
      const bool ok = (unsigned)(r.iy0 + ki) < (unsigned)g.h && (unsigned)(r.ix0 + kj) < (unsigned)g.w;
      v[e] = ldg_or_zero(r.xr + t.x, ok);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 a_fix(int, int64_t, int, int64_t, const uint8_t*, float4 v) const { return relu4(v, relu); }
  __device__ float4 b_quad(int, int64_t n0, int row, int64_t k64, const uint8_t*) const {
    // (32-bit index math: every operand has < 2^31 elements, checked at launch)
    const int n = (int)n0 + row, k = (int)k64, Ni = (int)N, Ki = (int)K;
    if ((Ki & 3) == 0) return ldg4_or_zero(wt + (n * Ki + k), n < Ni && k < Ki);
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = ldg_or_zero(wt + (n * Ki + k + e), n < Ni && k + e < Ki);
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  DPG_NO_FIX(b_fix)
  __device__ void epilogue_row(int, int split, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    if (ksplit > 1) {
      float* out = part + ((int64_t)split * N + n0) * M + m;
      for (int j = 0; j < nv; ++j) out[j * M] = v[j];
      return;
    }
    uint32_t n, p;
    g.fP.divmod((uint32_t)m, n, p);
    float* out = y + (int64_t)n * g.oc * g.P + p;
    float val[16];
    for (int j = 0; j < nv; ++j) {
      val[j] = v[j] + (bias ? __ldg(bias + n0 + j) : 0.f);
      out[(n0 + j) * g.P] = val[j];
    }
    if (yh) {
      float* outh = yh + (int64_t)m * g.oc + n0;
      if (nv == 16 && (g.oc & 3) == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(outh + j) = make_float4(relu_if(val[j], relu_out), relu_if(val[j + 1], relu_out),
                                                             relu_if(val[j + 2], relu_out), relu_if(val[j + 3], relu_out));
      } else {
        for (int j = 0; j < nv; ++j) outh[j] = relu_if(val[j], relu_out);
      }
    }
  }
  __device__ void epilogue_cta(int, int, int, double) const {}
};

// sum_s part[s * stride + i] in split order, 8 independent loads in flight per round
__device__ __forceinline__ float sum_splits(const float* __restrict__ part, int ksplit, int64_t stride, int64_t i) {
  float acc = 0.f;
  int s = 0;
  for (; s + 8 <= ksplit; s += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(part + (int64_t)(s + u) * stride + i);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  for (; s < ksplit; ++s) acc += __ldg(part + (int64_t)s * stride + i);
  return acc;
}

// Y[n][oc][p] = bias[oc] + sum_s part[s][oc][n*P + p]
__global__ void fwd_reduce_kernel(const float* __restrict__ part, int ksplit, int64_t M, int64_t oc,
                                  int64_t P, const float* __restrict__ bias, float* __restrict__ y,
                                  float* __restrict__ yh, int relu_out) {
  pdl_wait();
  pdl_trigger();  // the next GEMM's CTAs may start their prologue beside this short pass
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // over oc * M, m fastest
  if (i >= oc * M) return;
  const int64_t c = i / M, m = i - c * M;
  const float acc = sum_splits(part, ksplit, oc * M, i);
  const int64_t n = m / P, p = m - n * P;
  const float val = acc + (bias ? bias[c] : 0.f);
  y[(n * oc + c) * P + p] = val;
  if (yh) yh[m * oc + c] = relu_if(val, relu_out);
}

size_t fwd_ws_bytes(const ConvGeom& cg) {
  const int ks = pick_ksplit(cg.b * cg.P(), cg.oc, cg.K(), 1);
  return ks > 1 ? sizeof(float) * (size_t)ks * (size_t)(cg.oc * cg.b * cg.P()) : 0;
}

void conv_fwd(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
              const ConvGeom& cg, float* y, void* ws, float* yh, int relu_out) {
  check_i32(cg);
  ConvFwd p;
  p.g = make_geo(cg);
  p.x = x; p.relu = x_relu; p.wt = w; p.bias = bias; p.y = y; p.yh = yh; p.relu_out = relu_out;
  p.M = cg.b * cg.P(); p.N = cg.oc; p.K = cg.K();
  p.ksplit = ws ? pick_ksplit(p.M, p.N, p.K, 1) : 1;
  p.part = static_cast<float*>(ws);
  p.scratch = (int)(8 * ((p.K + BK - 1) / BK) * BK + sizeof(ConvFwd::Row) * BM);
  launch_tc_auto(ctx, p, 1);
  if (p.ksplit > 1) {
    const int64_t n = p.M * p.N;
    ::dpg::launch_pdl(fwd_reduce_kernel, (unsigned)((n + 255) / 256), 256, 0, ctx->stream, p.part, p.ksplit, p.M, p.N, p.g.P, bias, y, yh, relu_out);
    DPG_LAUNCH_CHECK(ctx);
  }
}

// ------------------------------------------------------------------------------ dgrad
// One launch covers every stride-parity class (blockIdx.z = class). Inside class (ry, rx) the
// taps are ki = ry + s a, kj = rx + s c; for input pixel (iy, ix) of the class the output pixel of
// tap (a, c) is (oy0 - a, ox0 - c), oy0 = (iy + pad - ry) / s. k = (o, a, c).
constexpr int kMaxClasses = 16;
struct DClass {
  int ry, rx, iy0, ix0, hc, wc, nki, nkj;
  int64_t M, K;
};

struct ConvDgrad : TileRows {
  static constexpr bool kCtaReduce = false;
  Geo g;
  const float* dy;
  const float* wt;
  const float* mask;
  float* dx;
  float* part;  // split-K partials [ksplit][b*ic*h*w] (ksplit > 1)
  int64_t M, N, K, dx_numel;
  int ksplit, scratch, ncls;
  DClass cls[kMaxClasses];
  struct TEnt {  // (read back as one int2: {delta, a | c << 8 | o << 16})
    int delta;  // o*oh*ow - a*ow - c
    unsigned char a, c;
    short o;
  };
  struct Row {
    const float* dr;  // dy + (n, 0, oy0, ox0)
    int oy0, ox0;     // kBad-based for rows beyond the class (every bound check fails)
  };
  __device__ int64_t mdim(int z) const { return cls[z].M; }
  __device__ int64_t kdim(int z) const { return cls[z].K; }
  __device__ int ttab_bytes() const { return (int)(8 * ((K + BK - 1) / BK) * BK); }
  __device__ void setup(int z, int64_t m0, int64_t, uint8_t* s, int tid) const {
    const DClass& c = cls[z];
    TEnt* tt = reinterpret_cast<TEnt*>(s);
    Row* rows = reinterpret_cast<Row*>(s + ttab_bytes());
    const int taps = c.nki * c.nkj;
    const int kpad = (int)((c.K + BK - 1) / BK) * BK;
    for (int k = tid; k < kpad; k += kThreads) {
      if (k < c.K) {
        const int o = k / taps, t = k - o * taps;
        const int a = t / c.nkj, cc = t - a * c.nkj;
        tt[k] = TEnt{(o * g.oh - a) * g.ow - cc, (unsigned char)a, (unsigned char)cc, (short)o};
      } else {
        tt[k] = TEnt{0, (unsigned char)255, (unsigned char)255, (short)0};  // oy0 - 255 < 0: fails
      }
    }
    if (tid < BM) {
      Row r{dy, kBad, kBad};
      if (m0 + tid < c.M) {
        const int per = c.hc * c.wc;
        const int64_t m = m0 + tid;
        const int n = (int)(m / per), q = (int)(m - (int64_t)n * per);
        const int qy = q / c.wc, qx = q - qy * c.wc;
        const int iy = c.iy0 + g.stride * qy, ix = c.ix0 + g.stride * qx;
        const int oy0 = (iy + g.pad - c.ry) / g.stride, ox0 = (ix + g.pad - c.rx) / g.stride;
        r = Row{dy + (int64_t)n * g.oc * g.oh * g.ow + (int64_t)oy0 * g.ow + ox0, oy0, ox0};
      }
      rows[tid] = r;
    }
  }
  static constexpr bool kAQuadMajor = false;  // rows = input pixels of the class
  static constexpr bool kBQuadMajor = true;
  __device__ float4 a_quad(int, int64_t, int row, int64_t k, const uint8_t* s) const {
    const TEnt* tt = reinterpret_cast<const TEnt*>(s) + (int)k;
    const Row r = reinterpret_cast<const Row*>(s + ttab_bytes())[row];
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int2 t = *reinterpret_cast<const int2*>(tt + e);  // {delta, a | c << 8 | o << 16}
      const int ta = t.y & 0xff, tc = (t.y >> 8) & 0xff;
      const bool ok = (unsigned)(r.oy0 - ta) < (unsigned)g.oh && (unsigned)(r.ox0 - tc) < (unsigned)g.ow;
      v[e] = ldg_or_zero(r.dr + t.x, ok);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  DPG_NO_FIX(a_fix)
  __device__ float4 b_quad(int z, int64_t n0, int row, int64_t k64, const uint8_t* s) const {
    const DClass& c = cls[z];
    const TEnt* tt = reinterpret_cast<const TEnt*>(s);
    const int ch = (int)n0 + row, k = (int)k64, Kc = (int)c.K;
    const bool ch_ok = ch < (int)N;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int2 t = *reinterpret_cast<const int2*>(tt + k + e);  // (table padded to whole stages)
      const int ta = t.y & 0xff, tc = (t.y >> 8) & 0xff, to = t.y >> 16;
      const bool ok = ch_ok && k + e < Kc;
      v[e] = ldg_or_zero(wt + (((to * g.ic + ch) * g.kh + c.ry + g.stride * ta) * g.kw + c.rx + g.stride * tc), ok);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  DPG_NO_FIX(b_fix)
  __device__ void epilogue_row(int z, int split, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    const DClass& c = cls[z];
    const int per = c.hc * c.wc;
    const int n = (int)(m / per), q = (int)(m - (int64_t)n * per);
    const int qy = q / c.wc, qx = q - qy * c.wc;
    const int iy = c.iy0 + g.stride * qy, ix = c.ix0 + g.stride * qx;
    const int64_t hw = (int64_t)g.h * g.w;
    const int64_t base = (int64_t)n * g.ic * hw + (int64_t)iy * g.w + ix;
    if (ksplit > 1) {
      float* out = part + (int64_t)split * dx_numel;
      for (int j = 0; j < nv; ++j) out[base + (n0 + j) * hw] = v[j];
      return;
    }
    for (int j = 0; j < nv; ++j) {
      const int64_t off = base + (n0 + j) * hw;
      float val = v[j];
      if (mask && !(__ldg(mask + off) > 0.f)) val = 0.f;
      dx[off] = val;
    }
  }
  __device__ void epilogue_cta(int, int, int, double) const {}
};

// dx = mask ? (sum_s part[s]) : 0 (input-shaped partials; every class writes disjoint pixels)
__global__ void dgrad_reduce_kernel(const float* __restrict__ part, int ksplit, int64_t n,
                                    const float* __restrict__ mask, float* __restrict__ dx) {
  pdl_wait();
  pdl_trigger();  // the next GEMM's CTAs may start their prologue beside this short pass
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = sum_splits(part, ksplit, n, i);
  if (mask && !(mask[i] > 0.f)) acc = 0.f;
  dx[i] = acc;
}

static void dgrad_classes(const ConvGeom& cg, ConvDgrad& p) {
  const int s = (int)cg.stride;
  p.ncls = 0;
  p.M = 0;
  p.K = 0;
  for (int ry = 0; ry < s; ++ry)
    for (int rx = 0; rx < s; ++rx) {
      DClass c{};
      c.ry = ry; c.rx = rx;
      c.iy0 = ((ry - (int)cg.pad) % s + s) % s;
      c.ix0 = ((rx - (int)cg.pad) % s + s) % s;
      c.hc = c.iy0 < cg.h ? (int)((cg.h - c.iy0 + s - 1) / s) : 0;
      c.wc = c.ix0 < cg.w ? (int)((cg.w - c.ix0 + s - 1) / s) : 0;
      c.nki = ry < cg.kh ? (int)((cg.kh - ry + s - 1) / s) : 0;
      c.nkj = rx < cg.kw ? (int)((cg.kw - rx + s - 1) / s) : 0;
      c.M = cg.b * c.hc * c.wc;
      c.K = cg.oc * c.nki * c.nkj;
      p.cls[p.ncls++] = c;
      p.M = std::max(p.M, c.M);
      p.K = std::max(p.K, c.K);
    }
}

// (tap tables use a one-byte tap index with 255 as the out-of-range sentinel)
bool dgrad_supported(const ConvGeom& cg) {
  return cg.stride * cg.stride <= kMaxClasses && cg.oh < 255 && cg.ow < 255 && cg.kh < 255 && cg.kw < 255;
}

size_t dgrad_ws_bytes(const ConvGeom& cg) {
  ConvDgrad p;
  dgrad_classes(cg, p);
  const int ks = pick_ksplit(p.M, cg.ic, p.K, p.ncls);
  return ks > 1 ? sizeof(float) * (size_t)ks * (size_t)(cg.b * cg.ic * cg.h * cg.w) : 0;
}

void conv_dgrad(dpg_ctx* ctx, const float* dy, const float* w, const ConvGeom& cg,
                const float* mask_src, float* dx, void* ws) {
  check_i32(cg);
  ConvDgrad p;
  p.g = make_geo(cg);
  p.dy = dy; p.wt = w; p.mask = mask_src; p.dx = dx;
  dgrad_classes(cg, p);
  p.N = cg.ic;
  p.dx_numel = cg.b * cg.ic * cg.h * cg.w;
  p.ksplit = ws ? pick_ksplit(p.M, p.N, p.K, p.ncls) : 1;
  p.part = static_cast<float*>(ws);
  p.scratch = (int)(8 * ((p.K + BK - 1) / BK) * BK + sizeof(ConvDgrad::Row) * BM);
  // every input pixel lies in exactly one parity class and every (class, row tile, split) CTA
  // writes its rows (zeros when its K range is empty), so the partials need no clearing
  launch_tc_auto(ctx, p, p.ncls);
  if (p.ksplit > 1) {
    ::dpg::launch_pdl(dgrad_reduce_kernel, (unsigned)((p.dx_numel + 255) / 256), 256, 0, ctx->stream, p.part, p.ksplit, p.dx_numel, mask_src, dx);
    DPG_LAUNCH_CHECK(ctx);
  }
}

// ------------------------------------------------------------------------------ per-sample conv
struct ConvGs : TileRows {
  static constexpr bool kCtaReduce = true;
  Geo g;
  const float* x;
  int relu;
  const float* hw;
  float* gw;
  double* sq_part;
  int64_t M, N, K, bsz;
  int ksplit, scratch;
  struct Row {
    int plane;  // c*h*w
    short ki, kj;
  };
  __device__ int64_t mdim(int) const { return M; }
  __device__ int64_t kdim(int) const { return K; }
  __device__ void setup(int, int64_t m0, int64_t, uint8_t* s, int tid) const {
    PEnt* pt = reinterpret_cast<PEnt*>(s);
    Row* rows = reinterpret_cast<Row*>(s + ((4 * K + 15) & ~15));
    build_ptab(g, pt, tid);
    if (tid < BM && m0 + tid < M) {
      const int k = (int)(m0 + tid);
      const int khw = g.kh * g.kw;
      const int c = k / khw, r = k - c * khw;
      const int ki = r / g.kw, kj = r - ki * g.kw;
      rows[tid] = Row{c * g.h * g.w, (short)ki, (short)kj};
    }
  }
  static constexpr bool kAQuadMajor = true;  // rows = kcol; lanes walk positions
  static constexpr bool kBQuadMajor = true;  // highway rows contiguous in p
  __device__ float4 a_quad(int z, int64_t m0, int row, int64_t k64, const uint8_t* s) const {
    const PEnt* pt = reinterpret_cast<const PEnt*>(s);
    const int Ki = (int)K, k = (int)k64;
    const Row r = reinterpret_cast<const Row*>(s + ((4 * Ki + 15) & ~15))[row];
    const int base = z * (g.ic * g.h * g.w) + r.plane;  // < 2^31 (launch check)
    float v[4];
    if (k >= Ki) return make_float4(0.f, 0.f, 0.f, 0.f);
    PEnt t[4];
    ptab_quad(pt, k, t);  // k % 4 == 0; entries in [Ki, Ki rounded up to 4) are sentinels
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int iy = t[e].y + r.ki, ix = t[e].x + r.kj;
      const bool ok = (unsigned)iy < (unsigned)g.h && (unsigned)ix < (unsigned)g.w;
      v[e] = ldg_or_zero(x + (base + iy * g.w + ix), ok);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 a_fix(int, int64_t, int, int64_t, const uint8_t*, float4 v) const { return relu4(v, relu); }
  __device__ float4 b_quad(int z, int64_t n0, int row, int64_t k64, const uint8_t*) const {
    const int oc = (int)n0 + row, Ki = (int)K, k = (int)k64;
    const int h = (z * g.oc + oc) * Ki;
    if ((Ki & 3) == 0) return ldg4_or_zero(hw + (h + k), k < Ki);
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = ldg_or_zero(hw + (h + k + e), k + e < Ki);
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  DPG_NO_FIX(b_fix)
  __device__ void epilogue_row(int z, int, int64_t m, int64_t n0, const float* v, int nv, double& sq) const {
    float* out = gw ? gw + ((int64_t)z * g.oc + n0) * g.Kc + m : nullptr;
    for (int j = 0; j < nv; ++j) {
      if (out) st_stream(out + j * g.Kc, v[j]);
      sq += (double)v[j] * v[j];
    }
  }
  __device__ void epilogue_cta(int z, int, int tile_mn, double sq) const {
    if (sq_part) sq_part[(int64_t)tile_mn * bsz + z] = sq;
  }
};

int gs_conv_rows(const ConvGeom& cg) {
  return (int)(((cg.K() + BM - 1) / BM) * ((cg.oc + pick_bn(cg.oc) - 1) / pick_bn(cg.oc)));
}

void conv_gs(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const ConvGeom& cg,
             float* gw, double* sq_part) {
  check_i32(cg);
  ConvGs p;
  p.g = make_geo(cg);
  p.x = x; p.relu = x_relu; p.hw = hw; p.gw = gw; p.sq_part = sq_part;
  p.M = cg.K(); p.N = cg.oc; p.K = cg.P(); p.bsz = cg.b;
  p.ksplit = 1;
  p.scratch = (int)(((4 * p.K + 15) & ~15) + sizeof(ConvGs::Row) * BM);
  launch_tc_auto(ctx, p, cg.b);
}

// ------------------------------------------------------------------------------ clipped conv sum
struct ConvCsum : TileRows {
  static constexpr bool kCtaReduce = false;
  Geo g;
  const float* x;
  int relu;
  const float* hw;
  const float* scale;
  float* part;
  int64_t M, N, K, spl, bsz;
  int ksplit, scratch;
  struct Row {
    int plane;
    short ki, kj;
  };
  __device__ int64_t mdim(int) const { return M; }
  __device__ int64_t kdim(int) const { return K; }
  __device__ void setup(int, int64_t m0, int64_t, uint8_t* s, int tid) const {
    PEnt* pt = reinterpret_cast<PEnt*>(s);
    Row* rows = reinterpret_cast<Row*>(s + ((4 * g.P + 15) & ~15));
    build_ptab(g, pt, tid);
    if (tid < BM && m0 + tid < M) {
      const int k = (int)(m0 + tid);
      const int khw = g.kh * g.kw;
      const int c = k / khw, r = k - c * khw;
      const int ki = r / g.kw, kj = r - ki * g.kw;
      rows[tid] = Row{c * g.h * g.w, (short)ki, (short)kj};
    }
  }
  static constexpr bool kAQuadMajor = true;
  static constexpr bool kBQuadMajor = true;
  __device__ float4 a_quad(int z, int64_t m0, int row, int64_t k64, const uint8_t* s) const {
    const PEnt* pt = reinterpret_cast<const PEnt*>(s);
    const Row r = reinterpret_cast<const Row*>(s + ((4 * g.P + 15) & ~15))[row];
    const int k = (int)k64, Ki = (int)K, n_end = (int)bsz, chw = g.ic * g.h * g.w;
    float v[4];
    if ((g.P & 3) == 0) {
      // the quad's 4 k share one sample (k % 4 == 0, P % 4 == 0): one division, one base
      uint32_t qq, pp;
      g.fP.divmod((uint32_t)k, qq, pp);
      const int n = z * (int)spl + (int)qq;
      const float* xb = x + (n * chw + r.plane);
      const bool in = k < Ki && n < n_end;
      PEnt t4[4];
      ptab_quad(pt, (int)pp, t4);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const PEnt t = t4[e];
        const int iy = t.y + r.ki, ix = t.x + r.kj;
        const bool ok = in && (unsigned)iy < (unsigned)g.h && (unsigned)ix < (unsigned)g.w;
        v[e] = ldg_or_zero(xb + (iy * g.w + ix), ok);
      }
      return make_float4(v[0], v[1], v[2], v[3]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t qq, pp;
      g.fP.divmod((uint32_t)(k + e), qq, pp);
      const int n = z * (int)spl + (int)qq;
      const PEnt t = pt[pp];
      const int iy = t.y + r.ki, ix = t.x + r.kj;
      const bool ok = k + e < Ki && n < n_end && (unsigned)iy < (unsigned)g.h && (unsigned)ix < (unsigned)g.w;
      v[e] = ldg_or_zero(x + (n * chw + r.plane + iy * g.w + ix), ok);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 a_fix(int, int64_t, int, int64_t, const uint8_t*, float4 v) const { return relu4(v, relu); }
  // raw highway values; the clip scale s_n is applied when the stage is stored (b_fix)
  __device__ float4 b_quad(int z, int64_t n0, int row, int64_t k64, const uint8_t*) const {
    const int oc = (int)n0 + row, k = (int)k64, Ki = (int)K, n_end = (int)bsz, P = (int)g.P;
    if ((P & 3) == 0) {
      uint32_t qq, pp;
      g.fP.divmod((uint32_t)k, qq, pp);
      const int n = z * (int)spl + (int)qq;
      const bool ok = k < Ki && n < n_end;
      return ldg4_or_zero(hw + ((n * g.oc + oc) * P + (int)pp), ok);
    }
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t qq, pp;
      g.fP.divmod((uint32_t)(k + e), qq, pp);
      const int n = z * (int)spl + (int)qq;
      const bool ok = k + e < Ki && n < n_end;
      v[e] = ldg_or_zero(hw + ((n * g.oc + oc) * P + (int)pp), ok);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 b_fix(int z, int64_t, int, int64_t k64, const uint8_t*, float4 v) const {
    const int k = (int)k64, n_end = (int)bsz;
    if ((g.P & 3) == 0) {
      const int n = z * (int)spl + (int)g.fP.div((uint32_t)k);
      const float sc = ldg_or_zero(scale + n, n < n_end);
      return make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w);
    }
    float sc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int n = z * (int)spl + (int)g.fP.div((uint32_t)(k + e));
      sc[e] = ldg_or_zero(scale + n, n < n_end);
    }
    return make_float4(sc[0] * v.x, sc[1] * v.y, sc[2] * v.z, sc[3] * v.w);
  }
  __device__ void epilogue_row(int z, int, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    float* out = part + ((int64_t)z * g.oc + n0) * g.Kc + m;
    for (int j = 0; j < nv; ++j) out[j * g.Kc] = v[j];
  }
  __device__ void epilogue_cta(int, int, int, double) const {}
};

// CTAs the clipped-sum launches aim for (split count = this / output tiles; measured best: 3 per SM)
static int csum_ctas() { return 3 * kNumSMs; }

// Products one split accumulates in TMEM, at most. The tensor core's fp32 accumulation is not
// round-to-nearest: its error grows with the accumulation chain (measured, CIFAR conv2 clipped sum
// recomputed in fp64 from the device's own record: 1.4e-6 max-scaled at 256 products per split,
// 1.0e-5 at 1,792), so long sums (b = 4096) get more splits instead of longer chains.
constexpr int64_t kCsumChain = 512;

int csum_conv_splits(const ConvGeom& cg) {
  const int64_t tiles = ((cg.K() + BM - 1) / BM) * ((cg.oc + 127) / 128);
  int64_t splits = std::max((csum_ctas() + tiles - 1) / tiles, (cg.b * cg.P() + kCsumChain - 1) / kCsumChain);
  const int64_t max_by_k = std::max<int64_t>(1, (cg.b * cg.P()) / (2 * BK));
  splits = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(splits, cg.b), max_by_k));
  const int64_t spl = (cg.b + splits - 1) / splits;
  return (int)((cg.b + spl - 1) / spl);  // every split non-empty
}

void conv_csum(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const float* scale,
               const ConvGeom& cg, float* part, int splits) {
  check_i32(cg);
  ConvCsum p;
  p.g = make_geo(cg);
  p.x = x; p.relu = x_relu; p.hw = hw; p.scale = scale; p.part = part;
  p.spl = (cg.b + splits - 1) / splits;
  p.M = cg.K(); p.N = cg.oc; p.K = p.spl * cg.P(); p.bsz = cg.b;
  p.ksplit = 1;
  p.scratch = (int)(((4 * cg.P() + 15) & ~15) + sizeof(ConvCsum::Row) * BM);
  launch_tc_auto(ctx, p, splits);
}

// ------------------------------------------------------------------------------ linear, mid > 1
struct LinGs : TileRows {
  static constexpr bool kCtaReduce = true;
  const float* acts;
  int relu;
  const float* hw;
  float* gw;
  double* sq_part;
  int64_t M, N, K, bsz;  // M = d (i), N = r (o), K = mid
  int ksplit, scratch;
  __device__ int64_t mdim(int) const { return M; }
  __device__ int64_t kdim(int) const { return K; }
  __device__ void setup(int, int64_t, int64_t, uint8_t*, int) const {}
  static constexpr bool kAQuadMajor = false;  // rows = i contiguous
  static constexpr bool kBQuadMajor = false;  // rows = o contiguous
  __device__ float4 a_quad(int z, int64_t m0, int row, int64_t k64, const uint8_t*) const {
    const int i = (int)m0 + row, k = (int)k64, Ki = (int)K, Mi = (int)M;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = ldg_or_zero(acts + ((z * Ki + k + e) * Mi + i), k + e < Ki);
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 a_fix(int, int64_t, int, int64_t, const uint8_t*, float4 v) const { return relu4(v, relu); }
  __device__ float4 b_quad(int z, int64_t n0, int row, int64_t k64, const uint8_t*) const {
    const int o = (int)n0 + row, k = (int)k64, Ki = (int)K, Ni = (int)N;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = ldg_or_zero(hw + ((z * Ki + k + e) * Ni + o), k + e < Ki);
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  DPG_NO_FIX(b_fix)
  __device__ void epilogue_row(int z, int, int64_t m, int64_t n0, const float* v, int nv, double& sq) const {
    float* out = gw ? gw + ((int64_t)z * N + n0) * M + m : nullptr;
    for (int j = 0; j < nv; ++j) {
      if (out) st_stream(out + j * M, v[j]);
      sq += (double)v[j] * v[j];
    }
  }
  __device__ void epilogue_cta(int z, int, int tile_mn, double sq) const {
    if (sq_part) sq_part[(int64_t)tile_mn * bsz + z] = sq;
  }
};

int gs_linear_rows(int64_t d, int64_t r) {
  return (int)(((d + BM - 1) / BM) * ((r + pick_bn(r) - 1) / pick_bn(r)));
}

void linear_gs(dpg_ctx* ctx, const float* acts, int relu, const float* hw, int64_t b, int64_t mid,
               int64_t d, int64_t r, float* gw, double* sq_part) {
  check_i32_linear(b, mid, d, r);
  LinGs p{{}, acts, relu, hw, gw, sq_part, d, r, mid, b, 1, 0};
  launch_tc_auto(ctx, p, b);
}

struct LinCsum : TileRows {
  static constexpr bool kCtaReduce = false;
  const float* acts;
  int relu;
  const float* hw;
  const float* scale;
  float* part;
  int64_t M, N, K, spl, mid, bsz;
  int ksplit, scratch;
  FastDiv fmid;
  __device__ int64_t mdim(int) const { return M; }
  __device__ int64_t kdim(int) const { return K; }
  __device__ void setup(int, int64_t, int64_t, uint8_t*, int) const {}
  static constexpr bool kAQuadMajor = false;
  static constexpr bool kBQuadMajor = false;
  __device__ float4 a_quad(int z, int64_t m0, int row, int64_t k64, const uint8_t*) const {
    const int i = (int)m0 + row, k = (int)k64, Ki = (int)K, Mi = (int)M, midi = (int)mid;
    float v[4];
    if ((midi & 3) == 0) {  // the quad's 4 k are 4 consecutive t of one sample: one division
      uint32_t qq, t;
      fmid.divmod((uint32_t)k, qq, t);
      const int n = z * (int)spl + (int)qq;
      const float* base = acts + ((n * midi + (int)t) * Mi + i);
      const bool in = k < Ki && n < (int)bsz;
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = ldg_or_zero(base + e * Mi, in);
      return make_float4(v[0], v[1], v[2], v[3]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t qq, t;
      fmid.divmod((uint32_t)(k + e), qq, t);
      const int n = z * (int)spl + (int)qq;
      v[e] = ldg_or_zero(acts + ((n * midi + (int)t) * Mi + i), k + e < Ki && n < (int)bsz);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 a_fix(int, int64_t, int, int64_t, const uint8_t*, float4 v) const { return relu4(v, relu); }
  // raw highway values; the clip scale s_n is applied when the stage is stored (b_fix)
  __device__ float4 b_quad(int z, int64_t n0, int row, int64_t k64, const uint8_t*) const {
    const int o = (int)n0 + row, k = (int)k64, Ki = (int)K, Ni = (int)N, midi = (int)mid;
    float v[4];
    if ((midi & 3) == 0) {
      uint32_t qq, t;
      fmid.divmod((uint32_t)k, qq, t);
      const int n = z * (int)spl + (int)qq;
      const float* base = hw + ((n * midi + (int)t) * Ni + o);
      const bool in = k < Ki && n < (int)bsz;
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = ldg_or_zero(base + e * Ni, in);
      return make_float4(v[0], v[1], v[2], v[3]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t qq, t;
      fmid.divmod((uint32_t)(k + e), qq, t);
      const int n = z * (int)spl + (int)qq;
      v[e] = ldg_or_zero(hw + ((n * midi + (int)t) * Ni + o), k + e < Ki && n < (int)bsz);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ float4 b_fix(int z, int64_t, int, int64_t k, const uint8_t*, float4 v) const {
    if (((int)mid & 3) == 0) {  // one sample per quad: one scale
      const int64_t n = (int64_t)z * spl + fmid.div((uint32_t)k);
      const float sc = ldg_or_zero(scale + n, n < bsz);
      return make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w);
    }
    float sc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t n = (int64_t)z * spl + fmid.div((uint32_t)(k + e));
      sc[e] = ldg_or_zero(scale + n, n < bsz);
    }
    return make_float4(sc[0] * v.x, sc[1] * v.y, sc[2] * v.z, sc[3] * v.w);
  }
  __device__ void epilogue_row(int z, int, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    float* out = part + ((int64_t)z * N + n0) * M + m;
    for (int j = 0; j < nv; ++j) out[j * M] = v[j];
  }
  __device__ void epilogue_cta(int, int, int, double) const {}
};

int csum_linear_splits(int64_t b, int64_t mid, int64_t d, int64_t r) {
  const int64_t tiles = ((d + BM - 1) / BM) * ((r + 127) / 128);
  int64_t splits = std::max((csum_ctas() + tiles - 1) / tiles, (b * mid + kCsumChain - 1) / kCsumChain);
  const int64_t max_by_k = std::max<int64_t>(1, (b * mid) / (2 * BK));
  splits = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(splits, b), max_by_k));
  const int64_t spl = (b + splits - 1) / splits;
  return (int)((b + spl - 1) / spl);  // every split non-empty
}

void linear_csum(dpg_ctx* ctx, const float* acts, int relu, const float* hw, const float* scale,
                 int64_t b, int64_t mid, int64_t d, int64_t r, float* part, int splits) {
  check_i32_linear(b, mid, d, r);
  LinCsum p;
  p.acts = acts; p.relu = relu; p.hw = hw; p.scale = scale; p.part = part;
  p.spl = (b + splits - 1) / splits;
  p.M = d; p.N = r; p.K = p.spl * mid; p.mid = mid; p.bsz = b;
  p.ksplit = 1;
  p.scratch = 0;
  p.fmid = FastDiv((uint32_t)mid);
  launch_tc_auto(ctx, p, splits);
}

}  // namespace tc
}  // namespace dpg
