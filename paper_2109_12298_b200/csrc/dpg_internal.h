// dpg_internal.h — context, error plumbing and kernel launcher declarations shared by the
// libdpg.so translation units. Not part of the ABI (include/dpg.h is).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "dpg.h"

namespace dpg {

// C++ side of the error contract: thrown inside libdpg, caught at the ABI boundary and turned
// into a dpg_status (the reference's exception classes, errors.hpp:12-72).
struct Error : std::runtime_error {
  dpg_status code;
  Error(dpg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(dpg_status c, const std::string& m) { throw Error(c, m); }

#define DPG_CUDA(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      ::dpg::raise(DPG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));   \
  } while (0)

#define DPG_NCCL(expr)                                                                  \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess)                                                              \
      ::dpg::raise(DPG_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));   \
  } while (0)

// Device-side error record. Kernels that detect a reference error (non-finite per-sample
// gradient, out-of-range index / target) atomicMin a 64-bit key so the FIRST offender in the
// reference's execution order wins: stage (forward < loss < clip), then parameter / layer,
// then sample.
enum ErrStage : uint64_t {
  ERR_STAGE_EMBED_INDEX = 1,  // layers.hpp:425-426 (forward gather)
  ERR_STAGE_TARGET = 2,       // layers.hpp:905
  ERR_STAGE_NONFINITE = 3,    // optimizer.hpp:77-83
  ERR_STAGE_REMOTE = 4,       // another rank of the sample-sharded step reported an error
};
__host__ __device__ inline uint64_t err_key(uint64_t stage, uint64_t major, uint64_t sample) {
  return (stage << 56) | ((major & 0xFFFFFFull) << 32) | (sample & 0xFFFFFFFFull);
}
constexpr uint64_t ERR_NONE = ~0ull;

struct DeviceErr {
  unsigned long long key;  // ERR_NONE when clear
  unsigned long long aux;  // stage-specific detail (e.g. the raw index bits)
  unsigned int lock;       // report_error's writer lock (key and aux are updated together)
  unsigned int pad;
};

}  // namespace dpg

struct dpg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int64_t launches = 0;
  dpg::DeviceErr* dev_err = nullptr;  // device
  unsigned long long* clip_sync = nullptr;
  // device [2]: clip_factors' clipped count + CTA ticket (self-resetting) is clip_sync above
  uint64_t comm_gen = 0;  // bumped by dpg_ctx_init_comm: captured steps of an older communicator are stale
  dpg::DeviceErr* host_err = nullptr; // pinned mirror
  void* ws = nullptr;
  size_t ws_bytes = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool capturing = false;
  // streams owned by models of this context whose work a dpg_ctx_sync must also cover (the
  // pipelined host path's copy stream: loss read-backs)
  std::vector<cudaStream_t> extra_streams;

  // scratch space for operator-ABI calls (grows outside capture only)
  void* workspace(size_t bytes);
  // device-resident 0, 1, ..., n-1 (the identity row -> parameter map of an operator-ABI clip
  // factors call); grows outside capture only, so a call needs no host copy and no sync
  int32_t* iota = nullptr;
  int iota_n = 0;
  const int32_t* identity_rows(int n);
  // a side stream for independent work inside one operator-ABI call (e.g. a bias rule beside its
  // weight's rule): fork/join by events, so the call stays ordered on `stream` as a whole
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t main_saved = nullptr;
  bool can_fork();   // the side stream exists, or may be created now (no capture in progress)
  void fork_side();  // from here on, launches go to `side` (which waits for `stream`'s work so far)
  void end_side();   // launches go to `stream` again; the side work is marked for join_side()
  void join_side();  // `stream` waits for the side work

  // stage profiling (eager launches only): CUDA events on this stream around each stage,
  // with the stage's algorithmic bytes / flops
  struct ProfRec {
    std::string name;
    double bytes, flops;
    cudaEvent_t a, b;
    int64_t kernels = 0;  // launches inside the scope
    int64_t seq = 0;      // enqueue order of the scope
  };
  struct ProfAgg {
    double ms = 0, bytes = 0, flops = 0;
    int64_t count = 0, kernels = 0, first_seq = -1;
  };
  int64_t prof_seq = 0;
  bool profiling = false;
  // graph timeline (dpg_ctx_set_timeline): the stage scopes of a captured step become event-record
  // nodes on whichever stream (main or branch) runs them; after a replay each stage's start and
  // duration are read relative to the graph's first node, so the step's real overlap is visible
  bool timeline = false;
  cudaEvent_t tl_start = nullptr;
  std::vector<ProfRec> tl_recs;
  std::vector<ProfRec> prof_pending;
  std::map<std::string, ProfAgg> prof_agg;
  std::vector<cudaEvent_t> event_pool;
  std::string prof_text;
};

namespace dpg {

// Error-surfacing helpers (ctx.cpp). Reads the device error record (synchronising the stream),
// clears it, and throws the matching dpg::Error; `names` maps (stage, major) to a description of
// the offending layer / parameter in the reference's wording.
using ErrNamer = std::string (*)(const void* user, uint64_t stage, uint64_t major);
void throw_device_error(dpg_ctx* ctx, ErrNamer names, const void* user);
void sync_ctx(dpg_ctx* ctx);

// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the current device.
// Attributes are per (device, function), so the record is keyed on both and guarded by a mutex:
// several host threads may each drive their own GPU (one context per thread).
void ensure_smem_attr(const void* fn, int bytes);

inline void count_launch(dpg_ctx* ctx) { ++ctx->launches; }

// RAII stage timer: records an event pair on ctx->stream when profiling is on (never inside a
// graph capture). Kernel durations are read back by dpg_ctx_profile_read.
struct ProfScope {
  dpg_ctx* ctx;
  bool on;
  bool tl = false;  // timeline record (inside a capture)
  dpg_ctx::ProfRec rec;
  ProfScope(dpg_ctx* c, std::string name, double bytes, double flops);
  ~ProfScope();
};

std::string& thread_err();

// Run f, converting dpg::Error (and any other exception) into a status + message: no
// exception crosses the C ABI.
template <typename F>
dpg_status guard(dpg_ctx* ctx, F&& f) {
  try {
    f();
    return DPG_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what();
    thread_err() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    thread_err() = e.what();
    return DPG_ERR_INTERNAL;
  }
}

#define DPG_LAUNCH_CHECK(ctx)                                                            \
  do {                                                                                   \
    ::dpg::count_launch(ctx);                                                            \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      ::dpg::raise(DPG_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------------------
// Kernel launchers (implemented in the .cu files). All asynchronous on ctx->stream.
// Norm partials: `sq_part` is a [rows, b] double slab; a launcher writes `sq_rows(...)`
// consecutive rows starting at sq_part (row-major, stride b).
// ---------------------------------------------------------------------------------------

struct ConvGeom {
  int64_t b, ic, h, w, oc, kh, kw, stride, pad, oh, ow;
  int64_t K() const { return ic * kh * kw; }
  int64_t P() const { return oh * ow; }
};

// TMA-fed contractions (tg_conv.cu): NHWC activations / highways beside the NCHW buffers
struct TgPrepItem {
  const float* w;  // reference layout [O][C][kh][kw]
  float* wf;       // [O][kh][kw][C] (NHWC forward), nullable
  float* wd;       // [kh][kw][C][O] (dgrad), nullable
  int O, C, kh, kw;
};
struct TgPrepItems {
  TgPrepItem item[8];
  int count = 0;
};
namespace tg {
bool fwd_nhwc_ok(const ConvGeom& g);
bool dgrad_nhwc_ok(const ConvGeom& g);
void conv_fwd_nhwc(dpg_ctx* ctx, const float* xh, const float* wf, const float* bias, const ConvGeom& g, float* y,
                   float* yh, int relu_out);
void conv_dgrad_nhwc(dpg_ctx* ctx, const float* hh, const float* wd, const ConvGeom& g, const float* mask_h,
                     float* dx, float* dxh);
void prep_weights(dpg_ctx* ctx, const TgPrepItems& items);
// per-sample gradient + norm partials (3 rows) of a 3x3, 32-input-channel conv weight
bool rule_nhwc_ok(const ConvGeom& g);
void conv_rule_nhwc(dpg_ctx* ctx, const float* xh, const float* hw, const ConvGeom& g, float* gw, double* sq);
// clipped sum of a conv weight: MN-major NHWC input tiles, s ⊙ highway rows in TMEM
bool csum_nhwc_ok(const ConvGeom& g);
int csum_nhwc_splits(const ConvGeom& g);
void conv_csum_nhwc(dpg_ctx* ctx, const float* xh, const float* hw, const float* scale, const ConvGeom& g,
                    float* part, int splits);
void nchw_to_nhwc(dpg_ctx* ctx, const float* src, int relu, int64_t b, int64_t C, int64_t P, float* dst);
// T > 1 linear rule / clipped sum on the core (tg_linear.cu); DPG_TG=0 or DPG_TG_LIN=0: off
bool lin_shape_ok(int64_t b, int64_t mid, int64_t d, int64_t r);
bool lin_ok(const void* acts, const void* hw, const void* out, int64_t b, int64_t mid, int64_t d, int64_t r);
void lin_rule(dpg_ctx* ctx, const float* acts, int relu, const float* hw, int64_t b, int64_t mid, int64_t d,
              int64_t r, float* gw, double* sq_part);
int lin_csum_splits(int64_t b, int64_t mid, int64_t d, int64_t r);
void lin_csum(dpg_ctx* ctx, const float* acts, int relu, const float* hw, const float* scale, int64_t b,
              int64_t mid, int64_t d, int64_t r, float* part, int splits);
}  // namespace tg

namespace tc {
size_t fwd_ws_bytes(const ConvGeom& cg);
void conv_fwd(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
              const ConvGeom& cg, float* y, void* ws, float* yh = nullptr, int relu_out = 0);
bool dgrad_supported(const ConvGeom& cg);
size_t dgrad_ws_bytes(const ConvGeom& cg);
void conv_dgrad(dpg_ctx* ctx, const float* dy, const float* w, const ConvGeom& cg,
                const float* mask_src, float* dx, void* ws);
int gs_conv_rows(const ConvGeom& cg);
void conv_gs(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const ConvGeom& cg,
             float* gw, double* sq_part);
int csum_conv_splits(const ConvGeom& cg);
void conv_csum(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const float* scale,
               const ConvGeom& cg, float* part, int splits);
int gs_linear_rows(int64_t d, int64_t r);
void linear_gs(dpg_ctx* ctx, const float* acts, int relu, const float* hw, int64_t b, int64_t mid,
               int64_t d, int64_t r, float* gw, double* sq_part);
int csum_linear_splits(int64_t b, int64_t mid, int64_t d, int64_t r);
void linear_csum(dpg_ctx* ctx, const float* acts, int relu, const float* hw, const float* scale,
                 int64_t b, int64_t mid, int64_t d, int64_t r, float* part, int splits);
}  // namespace tc

namespace tk {  // thin-K conv layers (ic*kh*kw <= 64) on CUDA cores: rule (+ bias rule), clipped sum
bool supported(const ConvGeom& g);
void gs(dpg_ctx* ctx, const float* x, int relu, const float* hw, const ConvGeom& g, float* gw,
        double* sq_part, float* gb, double* sq_b, bool hw_nhwc = false);
int csum_splits(const ConvGeom& g);
void csum(dpg_ctx* ctx, const float* x, int relu, const float* hw, const float* scale,
          const ConvGeom& g, float* part, int splits, bool hw_nhwc = false);
}  // namespace tk

namespace rs {
bool supported(const ConvGeom& g);  // per-sample gradients, P <= 16
int gs_rows(const ConvGeom& g);
void gs(dpg_ctx* ctx, const float* x, int relu, const float* hw, const ConvGeom& g, float* gw,
        double* sq_part, float* gb = nullptr, double* sq_b = nullptr);
}  // namespace rs

// rules.cu — per-sample gradients
int sq_rows_linear(int64_t mid, int64_t d, int64_t r);
int sq_rows_conv2d(const ConvGeom& g, bool nhwc_rule = false);
int sq_rows_embedding(int64_t vocab, int64_t dim);
void launch_gs_linear(dpg_ctx* ctx, const float* acts, int acts_relu, const float* hw, int64_t b,
                      int64_t mid, int64_t d, int64_t r, float* gw, double* sq_part);
// gb / sq_b (optional): the bias rule fused into the same launch when gs_conv2d_fuses_bias(g)
// (sq_b then has sq_rows_conv2d_bias(g) rows), else a separate bias launch (one row)
void launch_gs_conv2d(dpg_ctx* ctx, const float* x, int x_relu, const float* hw, const ConvGeom& g,
                      float* gw, double* sq_part, float* gb = nullptr, double* sq_b = nullptr, bool hw_nhwc = false,
                      const float* xh = nullptr);
bool gs_conv2d_fuses_bias(const ConvGeom& g);
int sq_rows_conv2d_bias(const ConvGeom& g);
// bias rule: gb[n,o] = sum over middle of hw; `hw_layout_conv` selects [b, o, P] vs [b, mid, o]
void launch_gs_bias(dpg_ctx* ctx, const float* hw, int64_t b, int64_t mid, int64_t r,
                    bool hw_layout_conv, float* gb, double* sq_part);
// embedding: sort each sample's ids (validating them), then dense G and/or norms
void launch_embed_sort(dpg_ctx* ctx, const float* idx, int64_t b, int64_t t, int64_t vocab,
                       int32_t* sorted_v, int32_t* sorted_s);
void launch_gs_embedding(dpg_ctx* ctx, const int32_t* sorted_v, const int32_t* sorted_s,
                         const float* hw, int64_t b, int64_t t, int64_t vocab, int64_t dim,
                         float* g, double* sq_part);
// sum `rows` rows of a [rows, b] slab into out[b] (operator-ABI per-parameter norms)
void launch_sq_reduce(dpg_ctx* ctx, const double* part, int rows, int64_t b, double* out);

// clip.cu
void launch_clip_factors(dpg_ctx* ctx, const double* slab, const int32_t* row_param, int rows,
                         int64_t b, double c, double* norms, float* scale, int64_t* num_clipped);
size_t clipped_sum_ws_linear(int64_t b, int64_t mid, int64_t d, int64_t r);
size_t clipped_sum_ws_conv2d(const ConvGeom& g, bool nhwc_in = false);
void launch_clipped_sum_linear(dpg_ctx* ctx, const float* acts, int acts_relu, const float* hw,
                               const float* scale, int64_t b, int64_t mid, int64_t d, int64_t r,
                               float* sw, float* sb, int accumulate, void* ws);
void launch_clipped_sum_conv2d(dpg_ctx* ctx, const float* x, int x_relu, const float* hw,
                               const float* scale, const ConvGeom& g, float* sw, float* sb,
                               int accumulate, void* ws, bool hw_nhwc = false, const float* xh = nullptr);
size_t clipped_sum_ws_embedding(int64_t b, int64_t vocab);
void launch_clipped_sum_embedding(dpg_ctx* ctx, const int32_t* sorted_v, const int32_t* sorted_s,
                                  const float* hw, const float* scale, int64_t b, int64_t t,
                                  int64_t vocab, int64_t dim, float* summed, int accumulate,
                                  void* ws);
// Several small weighted sums over samples in one launch (the bias parameters of a model)
struct WsumItem {
  const float* g;  // [b, numel] per-sample values
  float* out;      // [numel]
  int64_t numel;
};
struct WsumItems {
  WsumItem item[16];
  int count;
};
void launch_wsum_multi(dpg_ctx* ctx, const WsumItems& items, const float* scale, int64_t b,
                       int accumulate);
void launch_sq_materialised(dpg_ctx* ctx, const float* g, int64_t b, int64_t numel,
                            double* sq_part);
int sq_rows_materialised(int64_t numel);
void launch_weighted_sum_materialised(dpg_ctx* ctx, const float* g, const float* scale, int64_t b,
                                      int64_t numel, float* summed, int accumulate);

// noise.cu
void launch_noise_update(dpg_ctx* ctx, float* params, const float* summed, float* grad, int64_t n,
                         double sigma, double c, double expected_batch, double lr, uint64_t seed,
                         uint64_t step, const float* injected, uint64_t* step_ptr,
                         unsigned long long* advance = nullptr, const float* status = nullptr);
// multi-rank steps: lane = error_pending ? 1 : 0, exchanged with the clipped sum (noise.cu)
void launch_status_lane(dpg_ctx* ctx, float* lane);
void launch_gaussian(dpg_ctx* ctx, float* out, int64_t n, double std_dev, uint64_t seed,
                     uint64_t step);
// the clipped-sum exchange over peer memory (noise.cu): rank r's optimizer arena mapped by every
// rank; flags[r] points at rank r's three 128-byte flag lines (signal, ack, local CTA counter)
constexpr int kMaxPeers = 8;
struct PeerSet {
  static constexpr int kSig = 0, kAck = 16, kCount = 32;  // in u64 units (128-byte lines)
  int world = 0, rank = 0;
  const float* summed[kMaxPeers] = {};
  unsigned long long* flags[kMaxPeers] = {};
};
void launch_noise_update_p2p(dpg_ctx* ctx, const PeerSet& ps, float* params, float* summed, float* reduced,
                             float* grad, int64_t n, double sigma, double c, double expected_batch, double lr,
                             uint64_t seed, uint64_t step, const float* injected, uint64_t* step_ptr,
                             unsigned long long* advance);

// layers.cu — supporting forward / backward
// ws: split-K scratch of at least conv_fwd_ws_bytes / conv_dgrad_ws_bytes (nullable: no split)
size_t conv_fwd_ws_bytes(const ConvGeom& g);
size_t conv_dgrad_ws_bytes(const ConvGeom& g);
void launch_conv2d_fwd(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
                       const ConvGeom& g, float* y, void* ws, float* yh = nullptr,
                       int relu_out = 0);
void launch_conv2d_dgrad(dpg_ctx* ctx, const float* dy, const float* w, const ConvGeom& g,
                         const float* mask_src, float* dx, void* ws);
// softmax-CE epilogue of the logits-producing linear forward (one row per sample)
struct LossFuse {
  const float* targets;
  float* loss;
  float* grad;
  int logits_relu;
  DeviceErr* err;
  // optional: the layer's input gradient in the same launch (dx = W^T grad, ReLU mask of the
  // previous layer's pre-activation folded in), bit-identical to launch_linear_dgrad's vector path
  float* dx = nullptr;
  const float* dmask = nullptr;
  // optional: dx also channels-last for a TMA-fed conv dgrad (flat j = c P + p -> [p][c])
  float* dx_nhwc = nullptr;
  int nhwc_c = 0, nhwc_p = 0;
};
// can the logits layer's forward launch also produce its input gradient (launch_linear_fwd + LossFuse::dx)?
bool linear_fwd_fuses_dgrad(int64_t d, int64_t r, const float* dx, const float* mask);
bool linear_fwd_fuses_loss(int64_t d, int64_t r, const float* x, const float* w);
void launch_linear_fwd(dpg_ctx* ctx, const float* x, int x_relu, const float* w, const float* bias,
                       int64_t rows, int64_t d, int64_t r, float* y, const LossFuse* loss = nullptr);
void launch_linear_dgrad(dpg_ctx* ctx, const float* dy, const float* w, int64_t rows, int64_t d,
                         int64_t r, const float* mask_src, float* dx);
void launch_embedding_fwd(dpg_ctx* ctx, const int32_t* sorted_v, const int32_t* sorted_s,
                          const float* table, int64_t b, int64_t t, int64_t dim, float* out);
void launch_softmax_ce(dpg_ctx* ctx, const float* logits, int logits_relu, const float* targets,
                       int64_t b, int64_t k, float* loss, float* grad);
void launch_relu_mask(dpg_ctx* ctx, float* g, const float* mask_src, int64_t n);

// norm.cu — layer_norm over [b, positions, m] (trailing m), group_norm over [b, C, spatial]
void launch_layer_norm_fwd(dpg_ctx* ctx, const float* x, int relu, const float* gamma, const float* beta,
                           int64_t b, int64_t positions, int64_t m, double eps, float* y, float* xhat,
                           float* inv_std);
void launch_layer_norm_dgrad(dpg_ctx* ctx, const float* gy, const float* gamma, const float* xhat,
                             const float* inv_std, int64_t b, int64_t positions, int64_t m,
                             const float* mask, float* gx);
void launch_group_norm_fwd(dpg_ctx* ctx, const float* x, int relu, const float* gamma, const float* beta,
                           int64_t b, int64_t channels, int64_t spatial, int64_t groups, double eps,
                           float* y, float* xhat, float* inv_std);
void launch_group_norm_dgrad(dpg_ctx* ctx, const float* gy, const float* gamma, const float* xhat,
                             const float* inv_std, int64_t b, int64_t channels, int64_t spatial,
                             int64_t groups, const float* mask, float* gx);
// per-sample gamma / beta records (either may be NULL) and their squared norms [b]
void launch_norm_rule(dpg_ctx* ctx, const float* hw, const float* xhat, int64_t b, int64_t channels,
                      int64_t positions, bool group_layout, float* gg, float* gb, double* sq_g, double* sq_b);

}  // namespace dpg
