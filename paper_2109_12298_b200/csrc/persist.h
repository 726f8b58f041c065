// persist.h — parameters of the persistent small-batch step kernel (persist.cu), filled by the
// engine (model.cpp).
#pragma once

#include <cstdint>

#include "dpg_internal.h"

namespace dpg {
namespace ps {

constexpr int kThreads = 512;
constexpr int kMaxLayers = 8;
constexpr int kMaxParams = 2 * kMaxLayers;

struct PLayer {
  int conv;            // 1 = conv2d, 0 = linear
  int in_relu;
  int C, H, W, O, KH, KW, S, PAD, OH, OW;  // conv geometry; linear: C = in, O = out
  int64_t in_numel, out_numel;
  const float* in;     // the model input (first layer)
  const float* w;      // parameters (reference layout)
  const float* bias;   // nullable
  float* gw;           // record block of the weight [b][numel_w]
  float* gb;           // record block of the bias [b][O], nullable
  int64_t numel_w;
  int in_s, out_s, hw_s, hw_prev_s;  // shared-memory offsets (floats) of the sample's tensors (-1: none)
  int pw;                            // parameter index of the weight (the bias is pw + 1)
};

struct Params {
  PLayer L[kMaxLayers];
  int nl;
  int64_t b;
  int out_relu;              // ReLU after the logits layer
  const float* targets;
  float* loss;               // nullable
  // clip / sum / update
  int np;
  const float* rec[kMaxParams];  // record block of parameter p
  int64_t numel[kMaxParams], off[kMaxParams];
  int64_t Ltot;
  double c;                  // max_grad_norm
  double* part;              // [np][b] per-(parameter, sample) squared norms
  double* norms;             // [b]
  float* scale;              // [b]
  long long* num_clipped;
  float* summed;
  float* grad;
  float* params;
  double std_dev;            // sigma * C
  float inv_e, lr;
  uint64_t seed, step;
  uint64_t* step_ptr;        // graph replays: the step lives on the device (and advances here)
  const float* injected;     // nullable
  DeviceErr* err;
  unsigned int* bar;         // grid barrier words [2] (zero between launches)
};

}  // namespace ps

// smem: bytes of the per-sample staging (max over layers of (input + output) floats)
void launch_persist_step(dpg_ctx* ctx, const ps::Params& p, int smem);

}  // namespace dpg
