// tc_conv.cu — the dense contractions of the step on tcgen05 (3xTF32, tc_gemm.cuh):
//
//   conv forward      Y[(n,p), oc]    = sum_kcol X~[n, kcol, p] W[oc, kcol]   (+ bias)
//   conv dgrad        dX[(n,pix), c]  = sum_(oc,tap) dY[n, oc, o(pix,tap)] W[oc, c, tap]
//                     per stride-parity class of input pixels (no wasted taps), ReLU mask fused
//   per-sample conv   G[n][oc][kcol]  = sum_p X~[n, kcol, p] B[n, oc, p]   + fused ||G_n||^2
//   clipped conv sum  S[oc][kcol]     = sum_(n,p) X~[n, kcol, p] (s_n B[n, oc, p])  (split-K)
//   per-sample linear G[n][o][i]      = sum_t A[n, t, i] B[n, t, o]           (mid > 1)
//   clipped linear    S[o][i]         = sum_(n,t) A[n, t, i] (s_n B[n, t, o])  (split-K)
//
// The GEMM row dimension (UMMA M = 128 TMEM lanes = epilogue threads) is always the dimension
// that is contiguous in the output, so the epilogue stores of a warp are coalesced.
#include "conv_common.cuh"
#include "tc_gemm.cuh"

namespace dpg {
namespace tc {

// im2col column decoder kcol -> (c, ki, kj) with fast division
struct KcolDec {
  FastDiv khw, kw;
  __device__ __forceinline__ void dec(uint32_t k, int& c, int& ki, int& kj) const {
    uint32_t q, r, a, b;
    khw.divmod(k, q, r);
    kw.divmod(r, a, b);
    c = (int)q;
    ki = (int)a;
    kj = (int)b;
  }
};

struct Geo {
  int ic, h, w, oc, kh, kw, stride, pad, oh, ow;
  int64_t P, Kc;
  KcolDec kd;
  FastDiv fow, fP;
};

inline Geo make_geo(const ConvGeom& g) {
  Geo r;
  r.ic = (int)g.ic; r.h = (int)g.h; r.w = (int)g.w; r.oc = (int)g.oc;
  r.kh = (int)g.kh; r.kw = (int)g.kw; r.stride = (int)g.stride; r.pad = (int)g.pad;
  r.oh = (int)g.oh; r.ow = (int)g.ow;
  r.P = g.P();
  r.Kc = g.K();
  r.kd.khw = FastDiv((uint32_t)(g.kh * g.kw));
  r.kd.kw = FastDiv((uint32_t)g.kw);
  r.fow = FastDiv((uint32_t)g.ow);
  r.fP = FastDiv((uint32_t)g.P());
  return r;
}

// ------------------------------------------------------------------------------ forward
struct ConvFwd {
  static constexpr bool kCtaReduce = false;
  Geo g;
  const float* x;
  int relu;
  const float* wt;
  const float* bias;
  float* y;
  int64_t M, N, K;
  struct RowA {
    int64_t base;
    int iy0, ix0;
  };
  struct RowB {
    const float* w;
  };
  __device__ RowA row_a(int, int64_t m) const {
    uint32_t n, p, oy, ox;
    g.fP.divmod((uint32_t)m, n, p);
    g.fow.divmod(p, oy, ox);
    return RowA{(int64_t)n * g.ic * g.h * g.w, (int)oy * g.stride - g.pad, (int)ox * g.stride - g.pad};
  }
  __device__ float a(const RowA& r, int, int64_t k) const {
    int c, ki, kj;
    g.kd.dec((uint32_t)k, c, ki, kj);
    const int iy = r.iy0 + ki, ix = r.ix0 + kj;
    if ((unsigned)iy >= (unsigned)g.h || (unsigned)ix >= (unsigned)g.w) return 0.f;
    return relu_if(__ldg(x + r.base + ((int64_t)c * g.h + iy) * g.w + ix), relu);
  }
  __device__ RowB row_b(int, int64_t n) const { return RowB{wt + n * g.Kc}; }
  __device__ float b(const RowB& r, int, int64_t k) const { return __ldg(r.w + k); }
  __device__ void epilogue_row(int, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    uint32_t n, p;
    g.fP.divmod((uint32_t)m, n, p);
    float* out = y + (int64_t)n * g.oc * g.P + p;
    for (int j = 0; j < nv; ++j) out[(n0 + j) * g.P] = v[j] + (bias ? __ldg(bias + n0 + j) : 0.f);
  }
  __device__ void epilogue_cta(int, double) const {}
};

void conv_fwd(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
              const ConvGeom& cg, float* y) {
  ConvFwd p;
  p.g = make_geo(cg);
  p.x = x; p.relu = x_relu; p.wt = w; p.bias = bias; p.y = y;
  p.M = cg.b * cg.P(); p.N = cg.oc; p.K = cg.K();
  launch_tc_auto(ctx, p, 1);
}

// ------------------------------------------------------------------------------ dgrad
struct ConvDgrad {
  static constexpr bool kCtaReduce = false;
  Geo g;
  const float* dy;
  const float* wt;
  const float* mask;
  float* dx;
  int64_t M, N, K;
  int ry, rx, hc, wc, nkj, iy0, ix0;
  FastDiv fcls, fwc, ftaps, fnkj, fs;
  struct RowA {
    int64_t dybase;
    int iy, ix;
  };
  struct RowB {
    int c;
  };
  __device__ RowA row_a(int, int64_t m) const {
    uint32_t n, q, qy, qx;
    fcls.divmod((uint32_t)m, n, q);
    fwc.divmod(q, qy, qx);
    return RowA{(int64_t)n * g.oc * g.oh * g.ow, iy0 + g.stride * (int)qy, ix0 + g.stride * (int)qx};
  }
  __device__ __forceinline__ void tap(int64_t k, int& o, int& ki, int& kj) const {
    uint32_t oo, t, a, c;
    ftaps.divmod((uint32_t)k, oo, t);
    fnkj.divmod(t, a, c);
    o = (int)oo;
    ki = ry + g.stride * (int)a;
    kj = rx + g.stride * (int)c;
  }
  __device__ float a(const RowA& r, int, int64_t k) const {
    int o, ki, kj;
    tap(k, o, ki, kj);
    const int ty = r.iy + g.pad - ki, tx = r.ix + g.pad - kj;
    if (ty < 0 || tx < 0) return 0.f;
    const int oy = (int)fs.div((uint32_t)ty), ox = (int)fs.div((uint32_t)tx);
    if (oy >= g.oh || ox >= g.ow) return 0.f;
    return __ldg(dy + r.dybase + ((int64_t)o * g.oh + oy) * g.ow + ox);
  }
  __device__ RowB row_b(int, int64_t n) const { return RowB{(int)n}; }
  __device__ float b(const RowB& r, int, int64_t k) const {
    int o, ki, kj;
    tap(k, o, ki, kj);
    return __ldg(wt + (((int64_t)o * g.ic + r.c) * g.kh + ki) * g.kw + kj);
  }
  __device__ void epilogue_row(int, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    uint32_t n, q, qy, qx;
    fcls.divmod((uint32_t)m, n, q);
    fwc.divmod(q, qy, qx);
    const int iy = iy0 + g.stride * (int)qy, ix = ix0 + g.stride * (int)qx;
    const int64_t hw = (int64_t)g.h * g.w;
    const int64_t base = (int64_t)n * g.ic * hw + (int64_t)iy * g.w + ix;
    for (int j = 0; j < nv; ++j) {
      const int64_t off = base + (n0 + j) * hw;
      float val = v[j];
      if (mask && !(__ldg(mask + off) > 0.f)) val = 0.f;
      dx[off] = val;
    }
  }
  __device__ void epilogue_cta(int, double) const {}
};

void conv_dgrad(dpg_ctx* ctx, const float* dy, const float* w, const ConvGeom& cg,
                const float* mask_src, float* dx) {
  const int s = (int)cg.stride;
  for (int ry = 0; ry < s; ++ry)
    for (int rx = 0; rx < s; ++rx) {
      ConvDgrad p;
      p.g = make_geo(cg);
      p.dy = dy; p.wt = w; p.mask = mask_src; p.dx = dx;
      p.ry = ry; p.rx = rx;
      p.iy0 = ((ry - (int)cg.pad) % s + s) % s;
      p.ix0 = ((rx - (int)cg.pad) % s + s) % s;
      p.hc = p.iy0 < cg.h ? (int)((cg.h - p.iy0 + s - 1) / s) : 0;
      p.wc = p.ix0 < cg.w ? (int)((cg.w - p.ix0 + s - 1) / s) : 0;
      const int nki = ry < cg.kh ? (int)((cg.kh - ry + s - 1) / s) : 0;
      p.nkj = rx < cg.kw ? (int)((cg.kw - rx + s - 1) / s) : 0;
      if (p.hc == 0 || p.wc == 0) continue;
      p.M = cg.b * p.hc * p.wc;
      p.N = cg.ic;
      p.K = cg.oc * nki * p.nkj;
      p.fcls = FastDiv((uint32_t)(p.hc * p.wc));
      p.fwc = FastDiv((uint32_t)p.wc);
      p.ftaps = FastDiv((uint32_t)std::max(1, nki * p.nkj));
      p.fnkj = FastDiv((uint32_t)std::max(1, p.nkj));
      p.fs = FastDiv((uint32_t)s);
      launch_tc_auto(ctx, p, 1);
    }
}

// ------------------------------------------------------------------------------ per-sample conv
struct ConvGs {
  static constexpr bool kCtaReduce = true;
  Geo g;
  const float* x;
  int relu;
  const float* hw;
  float* gw;
  double* sq_part;
  int64_t M, N, K, bsz;
  struct RowA {
    int64_t base;  // x offset of (n, c) plane
    int ki, kj;
  };
  struct RowB {
    const float* h;
  };
  __device__ RowA row_a(int z, int64_t m) const {
    int c, ki, kj;
    g.kd.dec((uint32_t)m, c, ki, kj);
    return RowA{((int64_t)z * g.ic + c) * g.h * g.w, ki - g.pad, kj - g.pad};
  }
  __device__ float a(const RowA& r, int, int64_t k) const {
    uint32_t oy, ox;
    g.fow.divmod((uint32_t)k, oy, ox);
    const int iy = (int)oy * g.stride + r.ki, ix = (int)ox * g.stride + r.kj;
    if ((unsigned)iy >= (unsigned)g.h || (unsigned)ix >= (unsigned)g.w) return 0.f;
    return relu_if(__ldg(x + r.base + (int64_t)iy * g.w + ix), relu);
  }
  __device__ RowB row_b(int z, int64_t n) const { return RowB{hw + ((int64_t)z * g.oc + n) * g.P}; }
  __device__ float b(const RowB& r, int, int64_t k) const { return __ldg(r.h + k); }
  __device__ void epilogue_row(int z, int64_t m, int64_t n0, const float* v, int nv, double& sq) const {
    float* out = gw ? gw + ((int64_t)z * g.oc + n0) * g.Kc + m : nullptr;
    for (int j = 0; j < nv; ++j) {
      if (out) st_stream(out + j * g.Kc, v[j]);
      sq += (double)v[j] * v[j];
    }
  }
  __device__ void epilogue_cta(int z, double sq) const {
    if (sq_part) sq_part[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * bsz + z] = sq;
  }
};

int gs_conv_rows(const ConvGeom& cg) {
  const int64_t bn = cg.oc <= 16 ? 16 : cg.oc <= 32 ? 32 : cg.oc <= 64 ? 64 : 128;
  return (int)(((cg.K() + BM - 1) / BM) * ((cg.oc + bn - 1) / bn));
}

void conv_gs(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const ConvGeom& cg,
             float* gw, double* sq_part) {
  ConvGs p;
  p.g = make_geo(cg);
  p.x = x; p.relu = x_relu; p.hw = hw; p.gw = gw; p.sq_part = sq_part;
  p.M = cg.K(); p.N = cg.oc; p.K = cg.P(); p.bsz = cg.b;
  launch_tc_auto(ctx, p, cg.b);
}

// ------------------------------------------------------------------------------ clipped conv sum
struct ConvCsum {
  static constexpr bool kCtaReduce = false;
  Geo g;
  const float* x;
  int relu;
  const float* hw;
  const float* scale;
  float* part;
  int64_t M, N, K, spl, bsz;
  struct RowA {
    int64_t cplane;  // c * h * w
    int ki, kj;
  };
  struct RowB {
    int oc;
  };
  __device__ RowA row_a(int, int64_t m) const {
    int c, ki, kj;
    g.kd.dec((uint32_t)m, c, ki, kj);
    return RowA{(int64_t)c * g.h * g.w, ki - g.pad, kj - g.pad};
  }
  __device__ float a(const RowA& r, int z, int64_t k) const {
    uint32_t q, p, oy, ox;
    g.fP.divmod((uint32_t)k, q, p);
    const int64_t n = (int64_t)z * spl + q;
    if (n >= bsz) return 0.f;
    g.fow.divmod(p, oy, ox);
    const int iy = (int)oy * g.stride + r.ki, ix = (int)ox * g.stride + r.kj;
    if ((unsigned)iy >= (unsigned)g.h || (unsigned)ix >= (unsigned)g.w) return 0.f;
    return relu_if(__ldg(x + n * g.ic * g.h * g.w + r.cplane + (int64_t)iy * g.w + ix), relu);
  }
  __device__ RowB row_b(int, int64_t n) const { return RowB{(int)n}; }
  __device__ float b(const RowB& r, int z, int64_t k) const {
    uint32_t q, p;
    g.fP.divmod((uint32_t)k, q, p);
    const int64_t n = (int64_t)z * spl + q;
    if (n >= bsz) return 0.f;
    return __ldg(scale + n) * __ldg(hw + (n * g.oc + r.oc) * g.P + p);
  }
  __device__ void epilogue_row(int z, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    float* out = part + ((int64_t)z * g.oc + n0) * g.Kc + m;
    for (int j = 0; j < nv; ++j) out[j * g.Kc] = v[j];
  }
  __device__ void epilogue_cta(int, double) const {}
};

int csum_conv_splits(const ConvGeom& cg) {
  const int64_t tiles = ((cg.K() + BM - 1) / BM) * ((cg.oc + 127) / 128);
  // ~2 CTAs per SM, at least 2 k-stages of work per split
  int64_t splits = (2 * kNumSMs + tiles - 1) / tiles;
  const int64_t max_by_k = std::max<int64_t>(1, (cg.b * cg.P()) / (2 * BK));
  splits = std::min<int64_t>(std::min<int64_t>(splits, cg.b), max_by_k);
  return (int)std::max<int64_t>(1, splits);
}

void conv_csum(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const float* scale,
               const ConvGeom& cg, float* part, int splits) {
  ConvCsum p;
  p.g = make_geo(cg);
  p.x = x; p.relu = x_relu; p.hw = hw; p.scale = scale; p.part = part;
  p.spl = (cg.b + splits - 1) / splits;
  p.M = cg.K(); p.N = cg.oc; p.K = p.spl * cg.P(); p.bsz = cg.b;
  launch_tc_auto(ctx, p, splits);
}

// ------------------------------------------------------------------------------ linear, mid > 1
struct LinGs {
  static constexpr bool kCtaReduce = true;
  const float* acts;
  int relu;
  const float* hw;
  float* gw;
  double* sq_part;
  int64_t M, N, K, bsz;  // M = d (i), N = r (o), K = mid
  struct RowA {
    int64_t i;
  };
  struct RowB {
    int64_t o;
  };
  __device__ RowA row_a(int, int64_t m) const { return RowA{m}; }
  __device__ float a(const RowA& r, int z, int64_t k) const {
    return relu_if(__ldg(acts + ((int64_t)z * K + k) * M + r.i), relu);
  }
  __device__ RowB row_b(int, int64_t n) const { return RowB{n}; }
  __device__ float b(const RowB& r, int z, int64_t k) const { return __ldg(hw + ((int64_t)z * K + k) * N + r.o); }
  __device__ void epilogue_row(int z, int64_t m, int64_t n0, const float* v, int nv, double& sq) const {
    float* out = gw ? gw + ((int64_t)z * N + n0) * M + m : nullptr;
    for (int j = 0; j < nv; ++j) {
      if (out) st_stream(out + j * M, v[j]);
      sq += (double)v[j] * v[j];
    }
  }
  __device__ void epilogue_cta(int z, double sq) const {
    if (sq_part) sq_part[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * bsz + z] = sq;
  }
};

int gs_linear_rows(int64_t d, int64_t r) {
  const int64_t bn = r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : 128;
  return (int)(((d + BM - 1) / BM) * ((r + bn - 1) / bn));
}

void linear_gs(dpg_ctx* ctx, const float* acts, int relu, const float* hw, int64_t b, int64_t mid,
               int64_t d, int64_t r, float* gw, double* sq_part) {
  LinGs p{acts, relu, hw, gw, sq_part, d, r, mid, b};
  launch_tc_auto(ctx, p, b);
}

struct LinCsum {
  static constexpr bool kCtaReduce = false;
  const float* acts;
  int relu;
  const float* hw;
  const float* scale;
  float* part;
  int64_t M, N, K, spl, mid, bsz;
  FastDiv fmid;
  struct RowA {
    int64_t i;
  };
  struct RowB {
    int64_t o;
  };
  __device__ RowA row_a(int, int64_t m) const { return RowA{m}; }
  __device__ float a(const RowA& r, int z, int64_t k) const {
    uint32_t q, t;
    fmid.divmod((uint32_t)k, q, t);
    const int64_t n = (int64_t)z * spl + q;
    if (n >= bsz) return 0.f;
    return relu_if(__ldg(acts + (n * mid + t) * M + r.i), relu);
  }
  __device__ RowB row_b(int, int64_t n) const { return RowB{n}; }
  __device__ float b(const RowB& r, int z, int64_t k) const {
    uint32_t q, t;
    fmid.divmod((uint32_t)k, q, t);
    const int64_t n = (int64_t)z * spl + q;
    if (n >= bsz) return 0.f;
    return __ldg(scale + n) * __ldg(hw + (n * mid + t) * N + r.o);
  }
  __device__ void epilogue_row(int z, int64_t m, int64_t n0, const float* v, int nv, double&) const {
    float* out = part + ((int64_t)z * N + n0) * M + m;
    for (int j = 0; j < nv; ++j) out[j * M] = v[j];
  }
  __device__ void epilogue_cta(int, double) const {}
};

int csum_linear_splits(int64_t b, int64_t mid, int64_t d, int64_t r) {
  const int64_t tiles = ((d + BM - 1) / BM) * ((r + 127) / 128);
  int64_t splits = (2 * kNumSMs + tiles - 1) / tiles;
  const int64_t max_by_k = std::max<int64_t>(1, (b * mid) / (2 * BK));
  splits = std::min<int64_t>(std::min<int64_t>(splits, b), max_by_k);
  return (int)std::max<int64_t>(1, splits);
}

void linear_csum(dpg_ctx* ctx, const float* acts, int relu, const float* hw, const float* scale,
                 int64_t b, int64_t mid, int64_t d, int64_t r, float* part, int splits) {
  LinCsum p;
  p.acts = acts; p.relu = relu; p.hw = hw; p.scale = scale; p.part = part;
  p.spl = (b + splits - 1) / splits;
  p.M = d; p.N = r; p.K = p.spl * mid; p.mid = mid; p.bsz = b;
  p.fmid = FastDiv((uint32_t)mid);
  launch_tc_auto(ctx, p, splits);
}

}  // namespace tc
}  // namespace dpg
