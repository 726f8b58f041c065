// conv_common.cuh — implicit im2col gather shared by the conv kernels.
#pragma once

#include "dpg_device.cuh"

namespace dpg {

// X~[n, kcol, p] of detail::im2col (layers.hpp:290-324) read straight from x[b, ic, h, w]:
// kcol = (c*kh + ki)*kw + kj, p = oy*ow + ox, zero outside the padded image; optional ReLU of
// the stored pre-activation (the relu layer folded into its consumer).
struct Im2col {
  const float* x;
  int relu;
  int ic, h, w, kh, kw, stride, pad, ow;
  __device__ __forceinline__ float operator()(int64_t n, int kcol, int p) const {
    const int khw = kh * kw;
    const int c = kcol / khw, rr = kcol - c * khw;
    const int ki = rr / kw, kj = rr - ki * kw;
    const int oy = p / ow, ox = p - oy * ow;
    const int iy = oy * stride + ki - pad, ix = ox * stride + kj - pad;
    if (iy < 0 || iy >= h || ix < 0 || ix >= w) return 0.f;
    return relu_if(__ldg(x + ((n * ic + c) * h + iy) * (int64_t)w + ix), relu);
  }
};

inline Im2col make_im2col(const float* x, int relu, const ConvGeom& g) {
  return Im2col{x, relu, (int)g.ic, (int)g.h, (int)g.w, (int)g.kh, (int)g.kw, (int)g.stride, (int)g.pad, (int)g.ow};
}

}  // namespace dpg
