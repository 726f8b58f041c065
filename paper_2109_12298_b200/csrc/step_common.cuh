// step_common.cuh — device pieces shared by the multi-kernel step and the persistent small-batch
// step (persist.cu): the Philox4x32-10 noise stream with the reference's Box-Muller construction,
// and the softmax cross-entropy of one sample.
#pragma once

#include <cstdint>

#include "dpg_device.cuh"

namespace dpg {

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      key.x += W0;
      key.y += W1;
    }
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
  }
  return ctr;
}

__device__ __forceinline__ void normal_pair(uint64_t seed, uint64_t step, uint64_t q, double& z0,
                                            double& z1) {
  const uint4 r = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), (uint32_t)step,
                                           (uint32_t)(step >> 32)),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint64_t x = ((uint64_t)r.y << 32) | r.x;
  const uint64_t y = ((uint64_t)r.w << 32) | r.z;
  const double u1 = (double)((x >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(y >> 11) * 0x1.0p-53;
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  z0 = rad * c;
  z1 = rad * s;
}

// softmax cross-entropy (layers.hpp:894-919), in double like the reference; per-sample loss
// and d(loss_n)/d(logits_n) = p - onehot (not divided by b). Invalid targets report
// (stage TARGET, sample n). One warp per sample: lanes own classes, max and sum by a fixed
// shuffle tree (the fp64 sum is associated differently from the reference's loop; the float
// outputs agree to rounding).
// one warp: loss and logit gradient of sample n from its k logits in `row`
__device__ __forceinline__ void softmax_ce_warp(const float* row, int logits_relu, const float* __restrict__ targets,
                                                int64_t n, int64_t k, float* __restrict__ loss,
                                                float* __restrict__ grad, DeviceErr* err) {
  const int lane = threadIdx.x & 31;
  const double tv = (double)targets[n];
  int64_t cls = 0;
  if (!(tv >= 0.0) || tv != floor(tv) || tv >= (double)k) {
    if (lane == 0)
      report_error(err, err_key(ERR_STAGE_TARGET, 0, (uint64_t)n), (uint64_t)__float_as_uint(targets[n]));
  } else {
    cls = (int64_t)tv;
  }
  double mx = -INFINITY;
  for (int64_t j = lane; j < k; j += 32) {
    const double v = (double)relu_if(row[j], logits_relu);
    mx = mx < v ? v : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = mx < t ? t : mx;
  }
  double denom = 0.0;
  for (int64_t j = lane; j < k; j += 32) denom += exp((double)relu_if(row[j], logits_relu) - mx);
  denom = warp_sum(denom);
  const double log_denom = log(denom);
  if (loss && lane == 0)
    loss[n] = (float)(-((double)relu_if(row[cls], logits_relu) - mx - log_denom));
  for (int64_t j = lane; j < k; j += 32) {
    const float lv = relu_if(row[j], logits_relu);
    const double p = exp((double)lv - mx) / denom;
    float gv = (float)(p - (j == cls ? 1.0 : 0.0));
    if (logits_relu && !(row[j] > 0.f)) gv = 0.f;  // relu layer after the last linear
    grad[n * k + j] = gv;
  }
}

}  // namespace dpg
