/*
 * CPU restatement of the reference DP-SGD step (TEST INFRASTRUCTURE ONLY; see dpg_oracle.h).
 * Shared helpers plus two instantiations of dpg_oracle_impl.inc (float and double).
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dpg_oracle.h"

void dpgo_set_error(const char* msg);

static int fail(int code, const char* msg) {
  dpgo_set_error(msg);
  return code;
}

/* detail::conv_out_extent (layers.hpp:283-288) */
static int64_t conv_out_extent(int64_t in, int64_t kernel, int64_t stride, int64_t pad) {
  const int64_t padded = in + 2 * pad;
  if (padded < kernel) return 0;
  return (padded - kernel) / stride + 1;
}

/* Parameter shapes per layer in build_model order (layers.hpp:933-969). */
static int layer_params(const dpgo_layer* d, int64_t nums[2]) {
  switch (d->kind) {
    case DPGO_LINEAR:
      nums[0] = d->out_features * d->in_features;
      nums[1] = d->out_features;
      return d->has_bias ? 2 : 1;
    case DPGO_EMBEDDING:
      nums[0] = d->vocab_size * d->embedding_dim;
      return 1;
    case DPGO_CONV2D:
      nums[0] = d->out_channels * d->in_channels * d->kernel_h * d->kernel_w;
      nums[1] = d->out_channels;
      return d->has_bias ? 2 : 1;
    default:
      return 0;
  }
}

/* NamedParam names (layers.hpp:936-952). */
static const char* param_name(const dpgo_layer* d, int k) {
  if (d->kind == DPGO_EMBEDDING) return "table";
  return k == 0 ? "weight" : "bias";
}

#define REAL float
#define SFX _f32
#include "dpg_oracle_impl.inc"
#undef REAL
#undef SFX

#define REAL double
#define SFX _f64
#include "dpg_oracle_impl.inc"
#undef REAL
#undef SFX
