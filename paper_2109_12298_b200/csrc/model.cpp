// model.cpp — the engine ABI (include/dpg.h, part 2): a device-resident ModelGraph
// (layers.hpp:227-245) driven like GradSampleModule + DpOptimizer (optimizer.hpp:138-278,
// 359-381), with the reference's lifecycle and error contract.
//
// Step structure (no host synchronisation, graph-capturable):
//   forward_backward : forward (ReLU folded into consumers) -> softmax-CE -> reverse walk:
//                      rule(l) with fused norm partials, then dgrad(l) with the ReLU mask
//   step             : clip_factors -> clipped sums ((scale ⊙ B)^T A, or the record) ->
//                      [NCCL all-reduce of the flat clipped sum] -> noise + update
// Independent launches run on branches (aux streams forked from and joined back into the
// caller's stream, so a captured graph holds them as parallel nodes): rule(l) only needs
// highway(l), so the rules run beside the dgrad chain; the per-layer clipped sums are mutually
// independent (disjoint slices of `summed`, private split-K workspaces). Stage profiling keeps
// everything on one stream.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dpg_internal.h"
#include "persist.h"

using dpg::ConvGeom;
using dpg::guard;
using dpg::raise;

namespace {

struct ParamInfo {
  int layer, slot;
  int64_t numel, offset;
  int sq_row0, sq_rows;
  std::string name;
  bool is_bias;
};

struct LayerPlan {
  dpg_layer_desc d{};
  int kind = 0;
  // input activation: buffer index (-1 = model input), relu flag, per-sample numel
  int in_buf = -1;
  bool in_relu = false;
  int64_t in_numel = 0;
  int out_buf = -1;  // parametric layers own an output (pre-activation) buffer
  int64_t out_numel = 0;
  int param0 = -1, nparams = 0;
  ConvGeom g{};            // conv2d (b filled per call)
  int64_t mid = 1;         // linear: rows per sample
  int64_t tokens = 0;      // embedding
  int prev_param_layer = -1;  // previous parametric layer (whose output feeds this one)
  // layer_norm / group_norm: channels C, positions per (sample, channel) Q, statistics blocks
  // per sample; forward cache (layers.hpp:249-262): normalized input and inv_std
  int64_t norm_c = 0, norm_q = 0, stat_blocks = 0;
  float* xhat = nullptr;
  float* inv_std = nullptr;
  // TMA-fed contractions (tg_conv.cu). tg_fwd: 0 = register-gather kernels (thin first layers:
  // C % 16 != 0), 1 = NHWC implicit im2col (input copy xh). tg_dgrad: the input gradient from the
  // NHWC highway copy hh. The producers write these copies in their epilogues
  // (xh_by_prev / hh_by_next); otherwise a transpose launch fills them.
  int tg_fwd = 0;
  bool tg_dgrad = false;
  bool xh_by_prev = false, hh_by_next = false;
  bool tg_csum = false;  // clipped sum on the TMA core from xh (tg_conv.cu ConvCsumT)
  bool tg_rule = false;  // per-sample rule on the TMA core from xh (tg_conv.cu ConvRuleT)
  // the highway lives only channels-last (hh): written by the next layer's TMA-fed dgrad, read by
  // this layer's thin-K rule / clipped sum (a first layer: no dgrad of its own reads it)
  bool hw_nhwc = false;
  int next_param_layer = -1;
  float* xh = nullptr;    // [b][H][W][C] of the layer input (ReLU applied)
  float* hh = nullptr;    // [b][OH][OW][O] of the layer's highway
  float* wf = nullptr;    // [2][O][kh][kw][C] (TF32 hi, lo)
  float* wd = nullptr;    // [2][kh][kw][C][O]
};

// DPG_TG_CSUM=1: conv clipped sums on the TMA-fed core (read when a model is planned; opt-in:
// measured slower on the CIFAR step, DESIGN.md §6 negative results); DPG_TG_CSUM=L<i>,<j>,...:
// only the conv layers of those model indices
bool tg_csum_enabled(size_t layer) {
  const char* e = std::getenv("DPG_TG_CSUM");
  if (!e) return false;
  if (e[0] == '1') return true;
  if (e[0] != 'L') return false;
  for (const char* p = e + 1; *p;) {
    char* end = nullptr;
    const long v = std::strtol(p, &end, 10);
    if (end == p) break;
    if (v == (long)layer) return true;
    p = *end == ',' ? end + 1 : end;
  }
  return false;
}

// DPG_TG_RULE=1: the 3x3 / 32-channel per-sample conv rule on the TMA-fed core (read when a model
// is planned; opt-in: measured no faster than the register-gather rule)
bool tg_rule_enabled() {
  const char* e = std::getenv("DPG_TG_RULE");
  return e && e[0] == '1';
}

bool tg_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DPG_TG");
    return !(e && e[0] == '0');
  }();
  return on;
}

int64_t conv_out_extent(int64_t in, int64_t kernel, int64_t stride, int64_t pad) {
  const int64_t padded = in + 2 * pad;
  if (padded < kernel) return 0;
  return (padded - kernel) / stride + 1;
}

const char* kind_name(int k) {
  static const char* names[] = {"linear", "embedding", "conv2d", "layer_norm", "group_norm",
                                "relu", "flatten"};
  return (k >= 0 && k < 7) ? names[k] : "custom";
}

std::string shape_str(const std::vector<int64_t>& s, int64_t b = -1) {
  std::string out = "[";
  bool first = true;
  if (b >= 0) {
    out += std::to_string(b);
    first = false;
  }
  for (int64_t e : s) {
    if (!first) out += ", ";
    out += std::to_string(e);
    first = false;
  }
  return out + "]";
}

}  // namespace

struct dpg_model {
  dpg_ctx* ctx = nullptr;
  std::vector<LayerPlan> layers;
  std::vector<ParamInfo> params;
  std::vector<int64_t> in_shape;
  int64_t in_numel = 0, max_b = 0, L = 0, out_width = 0;
  int out_buf = -1;
  bool out_relu = false;
  int sq_rows = 0;
  int embed_layer = -1;
  int64_t embed_tokens = 0;
  // arena
  char* arena = nullptr;
  float* p_params = nullptr;
  std::vector<float*> bufs;      // per-parametric-layer outputs [max_b, out_numel]
  std::vector<float*> highways;  // same shapes
  int32_t* row_param = nullptr;
  int32_t* sorted_v = nullptr;
  int32_t* sorted_s = nullptr;
  float* logits_grad = nullptr;
  size_t ws_bytes = 0;
  void* ws = nullptr;            // fwd / dgrad split-K partials (main stream only)
  std::vector<void*> csum_ws;    // per layer: clipped-sum split-K partials (any branch)
  // branches: aux streams + a ring of fork/join events
  static constexpr int kAux = 2;
  cudaStream_t aux[kAux] = {nullptr, nullptr};
  bool aux_dirty[kAux] = {false, false};
  static constexpr int kEvents = 64;
  cudaEvent_t evs[kEvents] = {};
  int ev_next = 0;
  float* x_stage = nullptr;  // host-path staging
  float* y_stage = nullptr;
  float* loss = nullptr;
  // pipelined host path (dpg_train_step_host_async): two staging slots filled on a copy stream
  float* xs[2] = {nullptr, nullptr};
  float* ys[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaStream_t read_stream = nullptr;  // loss read-backs (a separate queue: H2D never waits on them)
  cudaEvent_t copied[2] = {nullptr, nullptr};   // slot's H2D done
  cudaEvent_t consumed[2] = {nullptr, nullptr}; // step that read the slot done
  float* losses[2] = {nullptr, nullptr};         // per-slot loss buffers: their D2H runs on the copy stream
  cudaEvent_t loss_read[2] = {nullptr, nullptr}; // that D2H done (the slot's next step may overwrite)
  int64_t async_calls = 0;
  unsigned int* persist_bar = nullptr;  // grid barrier words of the persistent small-batch step
};

struct dpg_optimizer {
  dpg_model* m = nullptr;
  dpg_optimizer_config cfg{};
  // device state
  char* arena = nullptr;
  float* summed = nullptr;
  float* grad = nullptr;
  float* record = nullptr;  // [max_b * L] when materialised, else bias-only scratch
  float* bias_scratch = nullptr;
  double* slab = nullptr;
  double* norms = nullptr;
  float* scale = nullptr;
  int64_t* num_clipped = nullptr;
  uint64_t* step_dev = nullptr;
  unsigned long long* step_tick = nullptr;  // ticket of the kernel that advances step_dev in a replay
  // step_dev == dev_step_next when dev_step_known: the previous replay advanced it on the device,
  // so the next replay needs no host-to-device copy of the step
  bool dev_step_known = false;
  uint64_t dev_step_next = 0;
  // clipped-sum exchange over peer memory (dpg_optimizer_set_peers): world = 0 when unused
  dpg::PeerSet peers;
  float* reduced = nullptr;               // [L] the rank-order sum, copied into summed at the end
  unsigned long long* xflags = nullptr;   // this rank's flag lines (PeerSet::flags[rank])
  std::vector<void*> peer_maps;           // IPC mappings of the peers' arenas
  // GradientState (optimizer.hpp:47-57)
  bool has_grad_sample = false, consumed = false, has_summed = false, has_grad = false;
  int64_t accumulated = 0;
  int64_t pending_b = 0, last_b = 0;
  uint64_t steps = 0;
  const float* injected = nullptr;
  // the pending batch's input must stay valid until its fold: the first layer's clipped sum
  // re-reads it, as the reference's forward cache keeps the input tensor (layers.hpp:249-256)
  const float* pending_x = nullptr;
  // CUDA graphs of the whole train step, per batch size
  struct Graph {
    int64_t b;
    const float* x;
    const float* y;
    float* loss;
    cudaGraphExec_t exec;
    int64_t kernels;  // kernels per replay (gpu_launches evidence)
    uint64_t last_use;
  };
  // Bounded LRU of instantiated step graphs: Poisson sampling gives a new physical batch size
  // almost every step, so a miss re-captures and updates the least recently used executable in
  // place (cudaGraphExecUpdate: same topology, new kernel arguments) instead of instantiating.
  static constexpr size_t kMaxGraphs = 8;
  std::vector<Graph> graphs;
  uint64_t graph_clock = 0;
  uint64_t graph_comm_gen = 0;  // ctx->comm_gen the cached graphs were captured under
  // pinned ring the graph replays read their Philox step from (a pageable source could make the
  // H2D wait for the stream); a slot is reused only after the copy that read it has executed
  static constexpr int kStepRing = 16;
  uint64_t* step_ring = nullptr;  // pinned host [kStepRing]
  cudaEvent_t ring_ev[kStepRing] = {};
  bool ring_used[kStepRing] = {};
};

namespace {

std::string err_namer(const void* user, uint64_t stage, uint64_t major) {
  const dpg_model* m = static_cast<const dpg_model*>(user);
  if (stage == dpg::ERR_STAGE_NONFINITE && major < m->params.size()) {
    const ParamInfo& p = m->params[major];
    return "layer " + std::to_string(p.layer) + " parameter '" + p.name + "'";
  }
  if (stage == dpg::ERR_STAGE_EMBED_INDEX && m->embed_layer >= 0)
    return " [0, " + std::to_string(m->layers[m->embed_layer].d.vocab_size) + ")";
  if (stage == dpg::ERR_STAGE_TARGET) return " [0, " + std::to_string(m->out_width) + ")";
  return std::string();
}

void surface(dpg_model* m) { dpg::throw_device_error(m->ctx, err_namer, m); }

bool branches_on(const dpg_model* m) { return m->aux[0] && !m->ctx->profiling; }

cudaEvent_t next_event(dpg_model* m) {
  cudaEvent_t e = m->evs[m->ev_next];
  m->ev_next = (m->ev_next + 1) % dpg_model::kEvents;
  return e;
}

// Enqueue f's launches on aux stream i, ordered after everything already on the caller's stream.
template <class F>
void on_branch(dpg_model* m, int i, F&& f) {
  dpg_ctx* ctx = m->ctx;
  if (i < 0 || !branches_on(m)) {
    f();
    return;
  }
  const cudaEvent_t e = next_event(m);
  DPG_CUDA(cudaEventRecord(e, ctx->stream));
  DPG_CUDA(cudaStreamWaitEvent(m->aux[i], e, 0));
  const cudaStream_t main = ctx->stream;
  ctx->stream = m->aux[i];
  m->aux_dirty[i] = true;
  try {
    f();
  } catch (...) {
    ctx->stream = main;
    throw;
  }
  ctx->stream = main;
}

// The caller's stream waits for every branch forked since the last join.
void join_branches(dpg_model* m) {
  for (int i = 0; i < dpg_model::kAux; ++i) {
    if (!m->aux_dirty[i]) continue;
    const cudaEvent_t e = next_event(m);
    DPG_CUDA(cudaEventRecord(e, m->aux[i]));
    DPG_CUDA(cudaStreamWaitEvent(m->ctx->stream, e, 0));
    m->aux_dirty[i] = false;
  }
}

// Parameter / record pointer of param p for batch b: the record packs [b, numel] blocks in
// (layer, slot) order (GradSampleRecord, grad_sample.hpp:20-33).
float* gs_ptr(dpg_optimizer* o, int p, int64_t b) {
  const ParamInfo& pi = o->m->params[p];
  if (o->cfg.materialise_grad_sample) return o->record + b * pi.offset;
  if (pi.is_bias) return o->bias_scratch + b * pi.offset;  // bias_scratch indexed like record
  return nullptr;
}

void forward_backward_impl(dpg_optimizer* o, const float* x, const float* targets, int64_t b,
                           float* loss) {
  dpg_model* m = o->m;
  dpg_ctx* ctx = m->ctx;
  float* P = m->p_params;
  auto act = [&](int buf) -> const float* { return buf < 0 ? x : m->bufs[buf]; };
  // ---- per-step weight layouts of the TMA-fed convolutions: on a branch, beside the first
  // layers' forward; joined before the first launch that reads them ----
  bool prep_pending = false;
  {
    dpg::TgPrepItems items;
    for (auto& lp : m->layers) {
      if (!lp.wf && !lp.wd) continue;
      if (items.count == 8) raise(DPG_ERR_DIMENSION, "more than 8 TMA-fed convolution layers");
      items.item[items.count++] = {P + m->params[lp.param0].offset, lp.wf, lp.wd, (int)lp.g.oc, (int)lp.g.ic,
                                   (int)lp.g.kh, (int)lp.g.kw};
    }
    if (items.count) {
      on_branch(m, 0, [&] {
        dpg::ProfScope ps(ctx, "prep.weights", 8.0 * 2 * 135306, 0.0);
        dpg::tg::prep_weights(ctx, items);
      });
      prep_pending = true;
    }
  }
  // ---- forward (layers.hpp:576-592) ----
  bool loss_done = false;  // softmax-CE fused into the logits-producing linear forward
  int hh_by_logits = -1;   // layer whose NHWC highway the logits launch wrote
  int dgrad_fused = -1;    // ... and that layer's input gradient too (its backward dgrad is skipped)
  for (size_t l = 0; l < m->layers.size(); ++l) {
    LayerPlan& lp = m->layers[l];
    if (lp.param0 < 0) continue;
    const float* in = act(lp.in_buf);
    const float* w = P + m->params[lp.param0].offset;
    const float* bias = lp.nparams > 1 ? P + m->params[lp.param0 + 1].offset : nullptr;
    float* out = m->bufs[lp.out_buf];
    const double io = 4.0 * b * (lp.in_numel + lp.out_numel);
    switch (lp.kind) {
      case DPG_LAYER_LINEAR: {
        dpg::ProfScope ps(ctx, "fwd.linear[" + std::to_string(l) + "]",
                          io + 4.0 * m->params[lp.param0].numel,
                          2.0 * b * lp.mid * lp.d.in_features * lp.d.out_features);
        const bool last = lp.out_buf == m->out_buf && lp.mid == 1 &&
                          dpg::linear_fwd_fuses_loss(lp.d.in_features, lp.d.out_features, in, w);
        dpg::LossFuse ce{targets, loss, m->highways[m->out_buf], m->out_relu ? 1 : 0, nullptr};
        if (last && lp.prev_param_layer >= 0) {
          // the backward's first input gradient (dgrad of this layer) in the same launch
          const LayerPlan& prev = m->layers[lp.prev_param_layer];
          float* dst = m->highways[prev.out_buf];
          const float* mask = lp.in_relu ? m->bufs[prev.out_buf] : nullptr;
          if (dpg::linear_fwd_fuses_dgrad(lp.d.in_features, lp.d.out_features, dst, mask)) {
            ce.dx = dst;
            ce.dmask = mask;
            dgrad_fused = l;
            if (prev.tg_dgrad && prev.kind == DPG_LAYER_CONV2D && prev.g.oc * prev.g.P() == lp.d.in_features) {
              ce.dx_nhwc = prev.hh;  // the conv's TMA-fed dgrad reads its highway channels-last
              ce.nhwc_c = (int)prev.g.oc;
              ce.nhwc_p = (int)prev.g.P();
              hh_by_logits = lp.prev_param_layer;
            }
          }
        }
        dpg::launch_linear_fwd(ctx, in, lp.in_relu, w, bias, b * lp.mid, lp.d.in_features,
                               lp.d.out_features, out, last ? &ce : nullptr);
        loss_done = loss_done || last;
        break;
      }
      case DPG_LAYER_CONV2D: {
        ConvGeom g = lp.g;
        g.b = b;
        // NHWC copy of this layer's output for a TMA-fed consumer (ReLU as the consumer applies it)
        float* yh = nullptr;
        int relu_out = 0;
        if (lp.next_param_layer >= 0) {
          const LayerPlan& nx = m->layers[lp.next_param_layer];
          if (nx.tg_fwd) {
            yh = nx.xh;
            relu_out = nx.in_relu ? 1 : 0;
          }
        }
        if (lp.tg_fwd && !lp.xh_by_prev) {
          dpg::ProfScope ps(ctx, "nhwc.x[" + std::to_string(l) + "]", 8.0 * b * lp.in_numel, 0.0);
          dpg::tg::nchw_to_nhwc(ctx, in, lp.in_relu, b, g.ic, g.h * g.w, lp.xh);
        }
        if (lp.tg_fwd && prep_pending) {
          join_branches(m);
          prep_pending = false;
        }
        dpg::ProfScope ps(ctx, "fwd.conv2d[" + std::to_string(l) + "]",
                          io + 4.0 * m->params[lp.param0].numel, 2.0 * b * g.oc * g.K() * g.P());
        if (lp.tg_fwd)
          dpg::tg::conv_fwd_nhwc(ctx, lp.xh, lp.wf, bias, g, out, yh, relu_out);
        else
          dpg::launch_conv2d_fwd(ctx, in, lp.in_relu, w, bias, g, out, m->ws, yh, relu_out);
        break;
      }
      case DPG_LAYER_LAYER_NORM:
      case DPG_LAYER_GROUP_NORM: {
        const bool gn = lp.kind == DPG_LAYER_GROUP_NORM;
        dpg::ProfScope ps(ctx, std::string(gn ? "fwd.group_norm[" : "fwd.layer_norm[") + std::to_string(l) + "]",
                          4.0 * b * (3 * lp.in_numel + lp.stat_blocks), 0.0);
        if (gn)
          dpg::launch_group_norm_fwd(ctx, in, lp.in_relu, w, bias, b, lp.norm_c, lp.norm_q, lp.stat_blocks,
                                     lp.d.eps, out, lp.xhat, lp.inv_std);
        else
          dpg::launch_layer_norm_fwd(ctx, in, lp.in_relu, w, bias, b, lp.norm_q, lp.norm_c, lp.d.eps, out,
                                     lp.xhat, lp.inv_std);
        break;
      }
      case DPG_LAYER_EMBEDDING: {
        dpg::ProfScope ps(ctx, "fwd.embedding[" + std::to_string(l) + "]",
                          4.0 * b * lp.tokens * (1 + 2 * lp.d.embedding_dim), 0.0);
        dpg::launch_embed_sort(ctx, in, b, lp.tokens, lp.d.vocab_size, m->sorted_v, m->sorted_s);
        dpg::launch_embedding_fwd(ctx, m->sorted_v, m->sorted_s, w, b, lp.tokens,
                                  lp.d.embedding_dim, out);
        break;
      }
    }
  }
  // ---- loss (layers.hpp:894-919) ----
  const float* logits = act(m->out_buf);
  float* g_last = m->highways[m->out_buf];  // highway of the last parametric layer
  if (!loss_done) {
    dpg::ProfScope ps(ctx, "loss.softmax_ce", 4.0 * b * (2 * m->out_width + 2), 0.0);
    dpg::launch_softmax_ce(ctx, logits, m->out_relu, targets, b, m->out_width, loss, g_last);
  }
  // ---- reverse walk (grad_sample.hpp:277-303) ----
  double* slab = o->slab;
  int rule_branch = 0;
  for (int l = (int)m->layers.size() - 1; l >= 0; --l) {
    LayerPlan& lp = m->layers[l];
    if (lp.param0 < 0) continue;
    const float* in = act(lp.in_buf);
    const float* hw = m->highways[lp.out_buf];
    const ParamInfo& pw = m->params[lp.param0];
    float* gw = gs_ptr(o, lp.param0, b);
    double* sq_w = slab + (int64_t)pw.sq_row0 * b;
    const std::string ls = "[" + std::to_string(l) + "]";
    const double gwrite = gw ? 4.0 * b * pw.numel : 0.0;
    // rules alternate between the two aux streams (each needs only its own highway), and a
    // separate bias rule runs on the other one
    const int rb = rule_branch++ & 1;
    auto bias_rule = [&](int64_t mid, int64_t r, bool conv_layout) {
      on_branch(m, rb ^ 1, [&] {
        const ParamInfo& pb = m->params[lp.param0 + 1];
        dpg::ProfScope ps(ctx, "gs.bias" + ls, 4.0 * b * (lp.out_numel + r), 0.0);
        dpg::launch_gs_bias(ctx, hw, b, mid, r, conv_layout, gs_ptr(o, lp.param0 + 1, b),
                            slab + (int64_t)pb.sq_row0 * b);
      });
    };
    struct { int64_t mid, r, conv; } pending_bias{0, 0, -1};  // a separate bias rule, forked below
    // the first parametric layer has no input gradient: once the last dgrad is issued the caller's
    // stream is idle, so its rule runs there (a branch may still be busy with the rule before it)
    on_branch(m, lp.prev_param_layer < 0 ? -1 : rb, [&] {
    switch (lp.kind) {
      case DPG_LAYER_LINEAR: {
        {
          dpg::ProfScope ps(ctx, "gs.linear" + ls, 4.0 * b * (lp.in_numel + lp.out_numel) + gwrite,
                            2.0 * b * lp.mid * lp.d.in_features * lp.d.out_features);
          dpg::launch_gs_linear(ctx, in, lp.in_relu, hw, b, lp.mid, lp.d.in_features,
                                lp.d.out_features, gw, sq_w);
        }
        if (lp.nparams > 1) pending_bias = {lp.mid, lp.d.out_features, 0};
        break;
      }
      case DPG_LAYER_CONV2D: {
        ConvGeom g = lp.g;
        g.b = b;
        {
          dpg::ProfScope ps(ctx, "gs.conv2d" + ls, 4.0 * b * (lp.in_numel + lp.out_numel) + gwrite,
                            2.0 * b * g.oc * g.K() * g.P());
          if (lp.nparams > 1 && dpg::gs_conv2d_fuses_bias(g)) {
            // bias rule in the same launch (its norm rows: one per oc tile)
            dpg::launch_gs_conv2d(ctx, in, lp.in_relu, lp.hw_nhwc ? lp.hh : hw, g, gw, sq_w,
                                  gs_ptr(o, lp.param0 + 1, b), slab + (int64_t)m->params[lp.param0 + 1].sq_row0 * b,
                                  lp.hw_nhwc);
            break;
          }
          dpg::launch_gs_conv2d(ctx, in, lp.in_relu, lp.hw_nhwc ? lp.hh : hw, g, gw, sq_w, nullptr, nullptr,
                                lp.hw_nhwc, lp.tg_rule ? lp.xh : nullptr);
        }
        if (lp.nparams > 1) pending_bias = {g.P(), g.oc, 1};
        break;
      }
      case DPG_LAYER_LAYER_NORM:
      case DPG_LAYER_GROUP_NORM: {
        const bool gn = lp.kind == DPG_LAYER_GROUP_NORM;
        const ParamInfo& pb = m->params[lp.param0 + 1];
        dpg::ProfScope ps(ctx, std::string(gn ? "gs.group_norm" : "gs.layer_norm") + ls,
                          4.0 * b * (2 * lp.out_numel + 2 * lp.norm_c), 0.0);
        dpg::launch_norm_rule(ctx, hw, lp.xhat, b, lp.norm_c, lp.norm_q, gn, gw, gs_ptr(o, lp.param0 + 1, b),
                              sq_w, slab + (int64_t)pb.sq_row0 * b);
        break;
      }
      case DPG_LAYER_EMBEDDING: {
        dpg::ProfScope ps(ctx, "gs.embedding" + ls, 4.0 * b * lp.out_numel + gwrite, 0.0);
        dpg::launch_gs_embedding(ctx, m->sorted_v, m->sorted_s, hw, b, lp.tokens,
                                 lp.d.vocab_size, lp.d.embedding_dim, gw, sq_w);
        break;
      }
    }
    });
    if (pending_bias.conv >= 0) bias_rule(pending_bias.mid, pending_bias.r, pending_bias.conv == 1);
    // input gradient for the previous parametric layer, with the ReLU mask folded in
    if (lp.prev_param_layer >= 0 && l != dgrad_fused) {
      const LayerPlan& prev = m->layers[lp.prev_param_layer];
      float* dst = m->highways[prev.out_buf];
      const float* mask = lp.in_relu ? m->bufs[prev.out_buf] : nullptr;
      const float* w = P + pw.offset;
      const double dio = 4.0 * (b * lp.out_numel + pw.numel + b * lp.in_numel * (mask ? 2 : 1));
      switch (lp.kind) {
        case DPG_LAYER_LINEAR: {
          dpg::ProfScope ps(ctx, "dgrad.linear" + ls, dio,
                            2.0 * b * lp.mid * lp.d.in_features * lp.d.out_features);
          dpg::launch_linear_dgrad(ctx, hw, w, b * lp.mid, lp.d.in_features, lp.d.out_features,
                                   mask, dst);
          break;
        }
        case DPG_LAYER_CONV2D: {
          ConvGeom g = lp.g;
          g.b = b;
          if (lp.tg_dgrad) {
            if (!lp.hh_by_next && hh_by_logits != l) {
              dpg::ProfScope ps(ctx, "nhwc.hw" + ls, 8.0 * b * lp.out_numel, 0.0);
              dpg::tg::nchw_to_nhwc(ctx, hw, 0, b, g.oc, g.P(), lp.hh);
            }
            dpg::ProfScope ps(ctx, "dgrad.conv2d" + ls, dio, 2.0 * b * g.oc * g.K() * g.P());
            // the previous layer's highway: NCHW (its rules / dgrad read it) and / or its NHWC copy
            dpg::tg::conv_dgrad_nhwc(ctx, lp.hh, lp.wd, g, lp.in_relu ? lp.xh : nullptr, prev.hw_nhwc ? nullptr : dst,
                                     (prev.tg_dgrad || prev.hw_nhwc) ? prev.hh : nullptr);
            break;
          }
          dpg::ProfScope ps(ctx, "dgrad.conv2d" + ls, dio, 2.0 * b * g.oc * g.K() * g.P());
          dpg::launch_conv2d_dgrad(ctx, hw, w, g, mask, dst, m->ws);
          break;
        }
        case DPG_LAYER_LAYER_NORM:
        case DPG_LAYER_GROUP_NORM: {
          const bool gn = lp.kind == DPG_LAYER_GROUP_NORM;
          dpg::ProfScope ps(ctx, std::string(gn ? "dgrad.group_norm" : "dgrad.layer_norm") + ls,
                            4.0 * b * (4 * lp.in_numel + lp.stat_blocks), 0.0);
          if (gn)
            dpg::launch_group_norm_dgrad(ctx, hw, w, lp.xhat, lp.inv_std, b, lp.norm_c, lp.norm_q,
                                         lp.stat_blocks, mask, dst);
          else
            dpg::launch_layer_norm_dgrad(ctx, hw, w, lp.xhat, lp.inv_std, b, lp.norm_q, lp.norm_c, mask, dst);
          break;
        }
        default:
          // embedding backward_input is zero (layers.hpp:626-629)
          DPG_CUDA(cudaMemsetAsync(dst, 0, sizeof(float) * b * prev.out_numel, ctx->stream));
      }
    }
  }
  join_branches(m);
}

// clip_and_sum of the pending batch into summed (fold_pending, optimizer.hpp:240-254)
void fold_impl(dpg_optimizer* o, int64_t b, const float* x) {
  dpg_model* m = o->m;
  dpg_ctx* ctx = m->ctx;
  const int accumulate = o->has_summed ? 1 : 0;
  {
    dpg::ProfScope ps(ctx, "clip_factors", 8.0 * m->sq_rows * b + 12.0 * b, 0.0);
    dpg::launch_clip_factors(ctx, o->slab, m->row_param, m->sq_rows, b, o->cfg.max_grad_norm,
                             o->norms, o->scale, o->num_clipped);
  }
  auto act = [&](int buf) -> const float* { return buf < 0 ? x : m->bufs[buf]; };
  // A weight's clipped sum comes from its stored per-sample gradients (the reference's own pass 2,
  // optimizer.hpp:99-114) when that record is smaller than the layer's activations + highway,
  // which (s ⊙ B)^T A would re-read (e.g. CIFAR conv1: 1.8 MB of G vs 23 MB of x and y);
  // otherwise from (s ⊙ B)^T A without touching G.
  std::vector<char> from_record(m->params.size(), 0);
  for (auto& lp : m->layers) {
    if (lp.param0 < 0) continue;
    for (int k = 0; k < lp.nparams; ++k) {
      const ParamInfo& pi = m->params[lp.param0 + k];
      from_record[lp.param0 + k] =
          pi.is_bias || (o->cfg.materialise_grad_sample && lp.kind != DPG_LAYER_EMBEDDING &&
                         2 * pi.numel < lp.in_numel + lp.out_numel);
    }
  }
  // stream plan for the per-layer (s ⊙ B)^T A launches: greedy, largest first, onto the least
  // loaded of aux 0 / aux 1 / the caller's stream, then the record weighted sums (one launch)
  // onto the least loaded. Estimated cost: a convolution's clipped sum is latency-bound at the
  // step's sizes (conv2..conv4 of CIFAR take 59-72 us in the graph timeline whatever their
  // flops), so a fixed part dominates; linear and embedding sums are short.
  double load[3] = {0.0, 0.0, 0.0};
  std::vector<int> stream_of(m->layers.size(), 2);
  {
    std::vector<std::pair<double, int>> cost;
    for (size_t l = 0; l < m->layers.size(); ++l) {
      const LayerPlan& lp = m->layers[l];
      if (lp.param0 < 0 || from_record[lp.param0]) continue;
      double fl = 0;
      if (lp.kind == DPG_LAYER_CONV2D) fl = 2.0 * b * lp.g.oc * lp.g.K() * lp.g.P();
      if (lp.kind == DPG_LAYER_LINEAR) fl = 2.0 * b * lp.mid * lp.d.in_features * lp.d.out_features;
      if (lp.kind == DPG_LAYER_EMBEDDING) fl = 8.0 * b * lp.out_numel;
      cost.push_back({(lp.kind == DPG_LAYER_CONV2D ? 20.0 : 2.0) + 5.0 * fl / 1e9, (int)l});
    }
    std::sort(cost.begin(), cost.end(), [](const auto& a, const auto& c) { return a.first > c.first; });
    for (auto& [c, l] : cost) {
      const int s = (int)(std::min_element(load, load + 3) - load);
      load[s] += c;
      stream_of[l] = s;
    }
  }
  const int record_stream = (int)(std::min_element(load, load + 3) - load);
  // record-based clipped sums (biases, normalisation affines, small weights): weighted column sums
  // of the per-sample records, all in one launch
  auto record_sums = [&] {
    if (!o->cfg.clipped_sum_from_record) {
      on_branch(m, record_stream < dpg_model::kAux ? record_stream : -1, [&] {
        dpg::WsumItems items{};
        double bytes = 0;
        for (auto& pi : m->params) {
          if (!from_record[&pi - &m->params[0]]) continue;
          if (items.count == 16) {
            dpg::launch_wsum_multi(ctx, items, o->scale, b, accumulate);
            items.count = 0;
          }
          items.item[items.count++] = {gs_ptr(o, (int)(&pi - &m->params[0]), b), o->summed + pi.offset, pi.numel};
          bytes += 4.0 * (b * pi.numel + 2 * pi.numel);
        }
        dpg::ProfScope ps(ctx, "csum.record[all]", bytes, 0.0);
        dpg::launch_wsum_multi(ctx, items, o->scale, b, accumulate);
      });
    }
  };
  // pass 0 forks the branches' launches, pass 1 enqueues the caller's stream's: a fork waits for
  // everything already on the caller's stream, so its long sums must come last
  int rr_branch = 0;
  for (int pass = 0; pass < 2; ++pass) {
  for (size_t l = 0; l < m->layers.size(); ++l) {
    LayerPlan& lp = m->layers[l];
    if (lp.param0 < 0) continue;
    for (int k = 0; k < lp.nparams; ++k) {
      const int p = lp.param0 + k;
      const ParamInfo& pi = m->params[p];
      float* dst = o->summed + pi.offset;
      float* rec = gs_ptr(o, p, b);
      const std::string ls = "[" + std::to_string(l) + "]";
      if (from_record[p] && !o->cfg.clipped_sum_from_record) continue;  // done above
      if (o->cfg.clipped_sum_from_record) {
        if (pass == 1) continue;
        // the reference's pass 2 over the stored per-sample gradients (exact order), one launch
        // per parameter, round-robin over the three streams
        on_branch(m, (rr_branch % 3) < dpg_model::kAux ? rr_branch % 3 : -1, [&] {
          dpg::ProfScope ps(ctx, std::string(pi.is_bias ? "csum.bias" : "csum.record") + ls,
                            4.0 * (b * pi.numel + 2 * pi.numel), 2.0 * b * pi.numel);
          dpg::launch_weighted_sum_materialised(ctx, rec, o->scale, b, pi.numel, dst, accumulate);
        });
        ++rr_branch;
        continue;
      }
      const float* in = act(lp.in_buf);
      const float* hw = m->highways[lp.out_buf];
      const double cio = 4.0 * (b * (lp.in_numel + lp.out_numel) + 2 * pi.numel);
      void* ws = m->csum_ws[l];
      const int br = stream_of[l];
      if ((br < dpg_model::kAux) != (pass == 0)) continue;
      on_branch(m, br < dpg_model::kAux ? br : -1, [&] {
      switch (lp.kind) {
        case DPG_LAYER_LINEAR: {
          dpg::ProfScope ps(ctx, "csum.linear" + ls, cio,
                            2.0 * b * lp.mid * lp.d.in_features * lp.d.out_features);
          dpg::launch_clipped_sum_linear(ctx, in, lp.in_relu, hw, o->scale, b, lp.mid,
                                         lp.d.in_features, lp.d.out_features, dst, nullptr,
                                         accumulate, ws);
          break;
        }
        case DPG_LAYER_CONV2D: {
          ConvGeom g = lp.g;
          g.b = b;
          dpg::ProfScope ps(ctx, "csum.conv2d" + ls, cio, 2.0 * b * g.oc * g.K() * g.P());
          dpg::launch_clipped_sum_conv2d(ctx, in, lp.in_relu, lp.hw_nhwc ? lp.hh : hw, o->scale, g, dst, nullptr,
                                         accumulate, ws, lp.hw_nhwc, lp.tg_csum ? lp.xh : nullptr);
          break;
        }
        case DPG_LAYER_EMBEDDING: {
          dpg::ProfScope ps(ctx, "csum.embedding" + ls, 4.0 * (b * lp.out_numel + 2 * pi.numel), 0.0);
          dpg::launch_clipped_sum_embedding(ctx, m->sorted_v, m->sorted_s, hw, o->scale, b,
                                            lp.tokens, lp.d.vocab_size, lp.d.embedding_dim, dst,
                                            accumulate, ws);
          break;
        }
      }
      });
    }
  }
  if (pass == 0 && record_stream < dpg_model::kAux) record_sums();
  }
  if (record_stream >= dpg_model::kAux) record_sums();
  join_branches(m);
  o->has_summed = true;
  o->accumulated += b;
  o->last_b = b;
}

// graph_mode: the Philox step is read from o->step_dev (graphs bake kernel arguments; the host
// writes the step there before each replay) and the host counter is advanced by the caller.
void finish_impl(dpg_optimizer* o, bool graph_mode) {
  dpg_model* m = o->m;
  dpg_ctx* ctx = m->ctx;
  // multi-rank: the status lane summed[L] travels with the clipped sum, so an error on any rank
  // skips the update on every rank (see noise.cu)
  if (o->peers.world > 1 || ctx->comm) dpg::launch_status_lane(ctx, o->summed + m->L);
  if (o->peers.world > 1) {
    dpg::ProfScope ps(ctx, "noise_update", 16.0 * m->L + 4.0 * o->peers.world * m->L, 0.0);
    dpg::launch_noise_update_p2p(ctx, o->peers, m->p_params, o->summed, o->reduced, o->grad, m->L,
                                 o->cfg.noise_multiplier, o->cfg.max_grad_norm, o->cfg.expected_batch_size,
                                 o->cfg.learning_rate, o->cfg.noise_seed, o->steps, o->injected,
                                 graph_mode ? o->step_dev : nullptr, graph_mode ? o->step_tick : nullptr);
    if (!graph_mode) {
      ++o->steps;
      o->dev_step_known = false;
    }
    o->has_grad = true;
    return;
  }
  if (ctx->comm) {
    dpg::ProfScope ps(ctx, "allreduce", 8.0 * m->L, 0.0);
    DPG_NCCL(ncclAllReduce(o->summed, o->summed, (size_t)m->L + 1, ncclFloat32, ncclSum, ctx->comm, ctx->stream));
  }
  dpg::ProfScope ps(ctx, "noise_update", 16.0 * m->L, 0.0);
  dpg::launch_noise_update(ctx, m->p_params, o->summed, o->grad, m->L, o->cfg.noise_multiplier,
                           o->cfg.max_grad_norm, o->cfg.expected_batch_size,
                           o->cfg.learning_rate, o->cfg.noise_seed, o->steps, o->injected,
                           graph_mode ? o->step_dev : nullptr, graph_mode ? o->step_tick : nullptr,
                           ctx->comm ? o->summed + m->L : nullptr);
  if (!graph_mode) {
    ++o->steps;
    o->dev_step_known = false;
  }
  o->has_grad = true;
}

// Lifecycle checks of set_grad_sample (optimizer.hpp:147-161)
void check_set_grad_sample(dpg_optimizer* o) {
  if (o->has_grad_sample && !o->consumed)
    raise(DPG_ERR_LIFECYCLE, "previous grad_sample was never consumed; call virtual_step or step first");
  if (o->has_grad) raise(DPG_ERR_LIFECYCLE, "grad from the last step is still present; call zero_grad first");
}

void step_impl(dpg_optimizer* o, const float* x, bool graph_mode) {
  if (o->has_grad) raise(DPG_ERR_LIFECYCLE, "step called twice without zero_grad in between");
  if (o->has_grad_sample && !o->consumed) {
    fold_impl(o, o->pending_b, x);
    o->consumed = true;
  }
  if (!o->has_summed)
    raise(DPG_ERR_LIFECYCLE,
          "step with no accumulated samples; run a backward or use step_empty_batch for a "
          "noise-only update");
  finish_impl(o, graph_mode);
}

void zero_grad_impl(dpg_optimizer* o) {
  o->has_grad_sample = false;
  o->consumed = false;
  o->has_summed = false;
  o->has_grad = false;
  o->accumulated = 0;
}

}  // namespace

extern "C" {

dpg_status dpg_model_create(dpg_ctx* ctx, const dpg_layer_desc* layers, int nlayers,
                            const int64_t* in_shape, int in_rank, int64_t max_batch,
                            dpg_model** out) {
  if (!out) return DPG_ERR_PARAMETER;
  *out = nullptr;
  dpg_model* m = new dpg_model();
  const dpg_status st = guard(ctx, [&] {
    if (!ctx) raise(DPG_ERR_PARAMETER, "null context");
    DPG_CUDA(cudaSetDevice(ctx->device));
    if (nlayers <= 0) raise(DPG_ERR_PARAMETER, "model needs at least one layer");
    if (max_batch <= 0) raise(DPG_ERR_PARAMETER, "max_batch must be positive");
    m->ctx = ctx;
    m->max_b = max_batch;
    m->in_shape.assign(in_shape, in_shape + in_rank);
    m->in_numel = 1;
    for (int64_t e : m->in_shape) m->in_numel *= e;
    // ---- shape walk (layer_forward checks, layers.hpp:382-573) ----
    std::vector<int64_t> shape = m->in_shape;
    int cur_buf = -1;
    bool cur_relu = false;
    int last_param_layer = -1;
    int64_t offset = 0;
    std::vector<int64_t> buf_numel;
    for (int l = 0; l < nlayers; ++l) {
      LayerPlan lp;
      lp.d = layers[l];
      lp.kind = lp.d.kind;
      int64_t numel = 1;
      for (int64_t e : shape) numel *= e;
      lp.in_buf = cur_buf;
      lp.in_relu = cur_relu;
      lp.in_numel = numel;
      auto shape_err = [&](const std::string& what) {
        raise(DPG_ERR_DIMENSION, "layer " + std::to_string(l) + " (" + kind_name(lp.kind) + "): " + what);
      };
      std::vector<std::pair<std::string, int64_t>> pshapes;
      switch (lp.kind) {
        case DPG_LAYER_LINEAR: {
          if (lp.d.in_features <= 0 || lp.d.out_features <= 0)
            raise(DPG_ERR_PARAMETER, "linear: feature counts must be positive");
          if (shape.empty() || shape.back() != lp.d.in_features)
            shape_err("expected trailing extent " + std::to_string(lp.d.in_features) + ", got input " +
                      shape_str(shape, 1));
          lp.mid = numel / lp.d.in_features;
          shape.back() = lp.d.out_features;
          pshapes.push_back({"weight", lp.d.out_features * lp.d.in_features});
          if (lp.d.has_bias) pshapes.push_back({"bias", lp.d.out_features});
          break;
        }
        case DPG_LAYER_EMBEDDING: {
          if (lp.d.vocab_size <= 0 || lp.d.embedding_dim <= 0)
            raise(DPG_ERR_PARAMETER, "embedding: extents must be positive");
          if (shape.size() != 1) shape_err("expected [batch, tokens] indices, got " + shape_str(shape, 1));
          if (l != 0 || cur_relu)
            raise(DPG_ERR_REGISTRY, "device embedding rule needs the embedding to read the model input");
          lp.tokens = shape[0];
          if (lp.tokens > 4096) shape_err("at most 4096 tokens per sample on device");
          shape = {lp.tokens, lp.d.embedding_dim};
          pshapes.push_back({"table", lp.d.vocab_size * lp.d.embedding_dim});
          m->embed_layer = l;
          m->embed_tokens = lp.tokens;
          break;
        }
        case DPG_LAYER_CONV2D: {
          const dpg_layer_desc& d = lp.d;
          if (d.in_channels <= 0 || d.out_channels <= 0 || d.kernel_h <= 0 || d.kernel_w <= 0 || d.stride <= 0)
            raise(DPG_ERR_PARAMETER, "conv2d: channel, kernel, and stride extents must be positive");
          if (shape.size() != 3 || shape[0] != d.in_channels)
            shape_err("expected [batch, " + std::to_string(d.in_channels) + ", h, w], got " + shape_str(shape, 1));
          const int64_t oh = conv_out_extent(shape[1], d.kernel_h, d.stride, d.padding);
          const int64_t ow = conv_out_extent(shape[2], d.kernel_w, d.stride, d.padding);
          if (oh == 0 || ow == 0) shape_err("kernel larger than padded input " + shape_str(shape, 1));
          lp.g = ConvGeom{0, d.in_channels, shape[1], shape[2], d.out_channels, d.kernel_h, d.kernel_w,
                          d.stride, d.padding, oh, ow};
          shape = {d.out_channels, oh, ow};
          pshapes.push_back({"weight", d.out_channels * d.in_channels * d.kernel_h * d.kernel_w});
          if (d.has_bias) pshapes.push_back({"bias", d.out_channels});
          break;
        }
        case DPG_LAYER_LAYER_NORM: {  // layers.hpp:468-506
          const dpg_layer_desc& d = lp.d;
          if (d.norm_size <= 0) raise(DPG_ERR_PARAMETER, "layer_norm: normalized shape must be non-empty");
          if (!(d.eps > 0.0)) raise(DPG_ERR_PARAMETER, "layer_norm: eps must be positive");
          if (shape.empty() || shape.back() != d.norm_size)
            shape_err("trailing dims of " + shape_str(shape, 1) + " do not match normalized shape [" +
                      std::to_string(d.norm_size) + "]");
          lp.norm_c = d.norm_size;
          lp.norm_q = numel / d.norm_size;
          lp.stat_blocks = lp.norm_q;
          pshapes.push_back({"gamma", d.norm_size});
          pshapes.push_back({"beta", d.norm_size});
          break;
        }
        case DPG_LAYER_GROUP_NORM: {  // layers.hpp:508-551
          const dpg_layer_desc& d = lp.d;
          if (d.groups <= 0 || d.norm_size <= 0 || d.norm_size % d.groups != 0)
            raise(DPG_ERR_PARAMETER, "group_norm: groups must be positive and divide channels");
          if (!(d.eps > 0.0)) raise(DPG_ERR_PARAMETER, "group_norm: eps must be positive");
          if (shape.empty() || shape[0] != d.norm_size)
            shape_err("expected [batch, " + std::to_string(d.norm_size) + ", ...], got " + shape_str(shape, 1));
          lp.norm_c = d.norm_size;
          lp.norm_q = numel / d.norm_size;
          lp.stat_blocks = d.groups;
          pshapes.push_back({"gamma", d.norm_size});
          pshapes.push_back({"beta", d.norm_size});
          break;
        }
        case DPG_LAYER_RELU:
          cur_relu = true;
          break;
        case DPG_LAYER_FLATTEN:
          shape = {numel};
          break;
        default:
          raise(DPG_ERR_REGISTRY, std::string("no device grad-sample rule registered for kind '") +
                                      kind_name(lp.kind) + "'");
      }
      if (!pshapes.empty()) {
        lp.param0 = (int)m->params.size();
        lp.nparams = (int)pshapes.size();
        for (size_t k = 0; k < pshapes.size(); ++k) {
          ParamInfo pi;
          pi.layer = l;
          pi.slot = (int)k;
          pi.numel = pshapes[k].second;
          pi.offset = offset;
          pi.name = pshapes[k].first;
          // biases and the normalisation affine parameters: small per-sample records whose clipped
          // sums are weighted sums of the records (launch_wsum_multi)
          pi.is_bias = pi.name == "bias" || lp.kind == DPG_LAYER_LAYER_NORM || lp.kind == DPG_LAYER_GROUP_NORM;
          offset += pi.numel;
          m->params.push_back(pi);
        }
        int64_t on = 1;
        for (int64_t e : shape) on *= e;
        lp.out_numel = on;
        lp.out_buf = (int)buf_numel.size();
        buf_numel.push_back(on);
        lp.prev_param_layer = last_param_layer;
        last_param_layer = l;
        cur_buf = lp.out_buf;
        cur_relu = false;
      }
      m->layers.push_back(lp);
    }
    if (last_param_layer < 0) raise(DPG_ERR_PARAMETER, "model has no trainable parameters");
    if (shape.size() != 1)
      raise(DPG_ERR_DIMENSION, "cross-entropy expects [batch, classes] logits, got " + shape_str(shape, 1));
    m->out_width = shape[0];
    m->out_buf = cur_buf;
    m->out_relu = cur_relu;
    m->L = offset;
    // the first parametric layer gets no input gradient (grad_sample.hpp:300)
    // ---- TMA-fed convolution plan ----
    for (size_t l = 0; l < m->layers.size(); ++l) {
      LayerPlan& lp = m->layers[l];
      if (lp.prev_param_layer >= 0) m->layers[lp.prev_param_layer].next_param_layer = (int)l;
      if (lp.kind != DPG_LAYER_CONV2D || !tg_enabled()) continue;
      if (dpg::tg::fwd_nhwc_ok(lp.g)) lp.tg_fwd = 1;
      lp.tg_dgrad = lp.tg_fwd && lp.prev_param_layer >= 0 && dpg::tg::dgrad_nhwc_ok(lp.g);
    }
    for (auto& lp : m->layers) {
      if (lp.kind == DPG_LAYER_CONV2D && lp.prev_param_layer < 0 && lp.next_param_layer >= 0 &&
          m->layers[lp.next_param_layer].tg_dgrad && dpg::tk::supported(lp.g))
        lp.hw_nhwc = true;
    }
    for (size_t l = 0; l < m->layers.size(); ++l) {
      LayerPlan& lp = m->layers[l];
      lp.tg_csum = lp.tg_fwd == 1 && !lp.hw_nhwc && dpg::tg::csum_nhwc_ok(lp.g) && tg_csum_enabled(l);
    }
    for (auto& lp : m->layers)
      lp.tg_rule = lp.tg_fwd == 1 && !lp.hw_nhwc && dpg::tg::rule_nhwc_ok(lp.g) && tg_rule_enabled();
    for (auto& lp : m->layers) {
      // every conv forward writes its consumer's NHWC copy in the epilogue
      if (lp.tg_fwd && lp.prev_param_layer >= 0) lp.xh_by_prev = m->layers[lp.prev_param_layer].kind == DPG_LAYER_CONV2D;
      if (lp.tg_dgrad && lp.next_param_layer >= 0) lp.hh_by_next = m->layers[lp.next_param_layer].tg_dgrad;
    }
    // ---- norm-partial rows (one row per producer output tile) ----
    int rows = 0;
    for (auto& lp : m->layers) {
      if (lp.param0 < 0) continue;
      for (int k = 0; k < lp.nparams; ++k) {
        ParamInfo& pi = m->params[lp.param0 + k];
        int r = 1;
        if (pi.is_bias && lp.kind == DPG_LAYER_CONV2D) r = dpg::sq_rows_conv2d_bias(lp.g);
        if (!pi.is_bias) {
          if (lp.kind == DPG_LAYER_LINEAR) r = dpg::sq_rows_linear(lp.mid, lp.d.in_features, lp.d.out_features);
          else if (lp.kind == DPG_LAYER_CONV2D) r = dpg::sq_rows_conv2d(lp.g, lp.tg_rule);
          else r = dpg::sq_rows_embedding(lp.d.vocab_size, lp.d.embedding_dim);
        }
        pi.sq_row0 = rows;
        pi.sq_rows = r;
        rows += r;
      }
    }
    m->sq_rows = rows;
    // ---- split-K workspaces: one for fwd / dgrad (main stream), one per layer for the clipped
    // sums (they run on concurrent branches); smaller batches may pick more splits, so each is
    // bounded over b = 1, 2, 4, ..., max_b and max_b ----
    size_t ws = 1 << 20;
    std::vector<size_t> csum_bytes(m->layers.size(), 0);
    for (size_t li = 0; li < m->layers.size(); ++li) {
      const LayerPlan& lp = m->layers[li];
      size_t& cs = csum_bytes[li];
      if (lp.kind == DPG_LAYER_LINEAR)
        for (int64_t bb = 1;; bb = std::min(bb * 2, max_batch)) {
          cs = std::max(cs, dpg::clipped_sum_ws_linear(bb, lp.mid, lp.d.in_features, lp.d.out_features));
          if (bb == max_batch) break;
        }
      if (lp.kind == DPG_LAYER_CONV2D) {
        ConvGeom g = lp.g;
        for (int64_t bb = 1;; bb = std::min(bb * 2, max_batch)) {
          g.b = bb;
          cs = std::max(cs, dpg::clipped_sum_ws_conv2d(g, lp.tg_csum));
          ws = std::max(ws, dpg::conv_fwd_ws_bytes(g));
          ws = std::max(ws, dpg::conv_dgrad_ws_bytes(g));
          if (bb == max_batch) break;
        }
      }
      if (lp.kind == DPG_LAYER_EMBEDDING) cs = std::max(cs, dpg::clipped_sum_ws_embedding(max_batch, lp.d.vocab_size));
    }
    m->ws_bytes = ws;
    // ---- arena ----
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t total = al(sizeof(float) * m->L);
    for (int64_t n : buf_numel) total += 2 * al(sizeof(float) * max_batch * n);
    total += al(sizeof(int32_t) * rows);
    total += 2 * al(sizeof(int32_t) * max_batch * std::max<int64_t>(1, m->embed_tokens));
    total += al(ws);
    for (size_t cs : csum_bytes) total += al(cs);
    total += 3 * (al(sizeof(float) * max_batch * m->in_numel) + al(sizeof(float) * max_batch));
    total += 3 * al(sizeof(float) * max_batch);
    for (auto& lp : m->layers)
      if (lp.stat_blocks) total += al(sizeof(float) * max_batch * lp.in_numel) + al(sizeof(float) * max_batch * lp.stat_blocks);
    auto tg_sizes = [&](const LayerPlan& lp, size_t* sz) {  // xh, hh, wf, wd
      const int64_t wn = lp.g.oc * lp.g.K();
      sz[0] = lp.tg_fwd == 1 ? sizeof(float) * max_batch * lp.in_numel : 0;
      sz[1] = (lp.tg_dgrad || lp.hw_nhwc) ? sizeof(float) * max_batch * lp.out_numel : 0;
      sz[2] = lp.tg_fwd == 1 ? 2 * sizeof(float) * wn : 0;  // TF32 hi and lo planes
      sz[3] = lp.tg_dgrad ? 2 * sizeof(float) * wn : 0;
    };
    for (auto& lp : m->layers) {
      size_t sz[4];
      tg_sizes(lp, sz);
      for (size_t z : sz) total += z ? al(z) : 0;
    }
    total += al(64);  // persist_bar
    DPG_CUDA(cudaMalloc(&m->arena, total));
    DPG_CUDA(cudaMemset(m->arena, 0, total));
    char* p = m->arena;
    auto take = [&](size_t bytes) {
      char* r = p;
      p += al(bytes);
      return r;
    };
    m->p_params = reinterpret_cast<float*>(take(sizeof(float) * m->L));
    for (int64_t n : buf_numel) {
      m->bufs.push_back(reinterpret_cast<float*>(take(sizeof(float) * max_batch * n)));
      m->highways.push_back(reinterpret_cast<float*>(take(sizeof(float) * max_batch * n)));
    }
    m->row_param = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * rows));
    m->sorted_v = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * max_batch * std::max<int64_t>(1, m->embed_tokens)));
    m->sorted_s = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * max_batch * std::max<int64_t>(1, m->embed_tokens)));
    m->ws = take(ws);
    for (size_t cs : csum_bytes) m->csum_ws.push_back(cs ? take(cs) : nullptr);
    for (auto& st : m->aux) DPG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& e : m->evs) DPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    m->x_stage = reinterpret_cast<float*>(take(sizeof(float) * max_batch * m->in_numel));
    m->y_stage = reinterpret_cast<float*>(take(sizeof(float) * max_batch));
    for (int q = 0; q < 2; ++q) {
      m->xs[q] = reinterpret_cast<float*>(take(sizeof(float) * max_batch * m->in_numel));
      m->ys[q] = reinterpret_cast<float*>(take(sizeof(float) * max_batch));
    }
    m->loss = reinterpret_cast<float*>(take(sizeof(float) * max_batch));
    for (auto& lb : m->losses) lb = reinterpret_cast<float*>(take(sizeof(float) * max_batch));
    for (auto& lp : m->layers)
      if (lp.stat_blocks) {
        lp.xhat = reinterpret_cast<float*>(take(sizeof(float) * max_batch * lp.in_numel));
        lp.inv_std = reinterpret_cast<float*>(take(sizeof(float) * max_batch * lp.stat_blocks));
      }
    m->persist_bar = reinterpret_cast<unsigned int*>(take(64));
    for (auto& lp : m->layers) {
      size_t sz[4];
      tg_sizes(lp, sz);
      float** dst[4] = {&lp.xh, &lp.hh, &lp.wf, &lp.wd};
      for (int q = 0; q < 4; ++q)
        if (sz[q]) *dst[q] = reinterpret_cast<float*>(take(sz[q]));
    }
    std::vector<int32_t> rp;
    for (size_t q = 0; q < m->params.size(); ++q)
      for (int r = 0; r < m->params[q].sq_rows; ++r) rp.push_back((int32_t)q);
    DPG_CUDA(cudaMemcpy(m->row_param, rp.data(), sizeof(int32_t) * rp.size(), cudaMemcpyHostToDevice));
  });
  if (st != DPG_OK) {
    if (m->arena) cudaFree(m->arena);
    delete m;
    return st;
  }
  *out = m;
  return DPG_OK;
}

void dpg_model_destroy(dpg_model* m) {
  if (!m) return;
  cudaSetDevice(m->ctx->device);
  cudaStreamSynchronize(m->ctx->stream);
  if (m->copy_stream) {
    cudaStreamSynchronize(m->copy_stream);
    cudaStreamSynchronize(m->read_stream);
    auto& xs = m->ctx->extra_streams;
    xs.erase(std::remove(xs.begin(), xs.end(), m->read_stream), xs.end());
    cudaStreamDestroy(m->copy_stream);
    cudaStreamDestroy(m->read_stream);
  }
  for (auto& st : m->aux)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  for (auto& e : m->evs)
    if (e) cudaEventDestroy(e);
  for (int q = 0; q < 2; ++q) {
    if (m->loss_read[q]) cudaEventDestroy(m->loss_read[q]);
    if (m->copied[q]) cudaEventDestroy(m->copied[q]);
    if (m->consumed[q]) cudaEventDestroy(m->consumed[q]);
  }
  if (m->arena) cudaFree(m->arena);
  delete m;
}

int64_t dpg_model_parameter_count(const dpg_model* m) { return m ? m->L : 0; }
int dpg_model_num_param_tensors(const dpg_model* m) { return m ? (int)m->params.size() : 0; }
int64_t dpg_model_output_width(const dpg_model* m) { return m ? m->out_width : 0; }
float* dpg_model_params(dpg_model* m) { return m ? m->p_params : nullptr; }

dpg_status dpg_model_param_info(const dpg_model* m, int p, int* layer, int* slot, int64_t* numel,
                                int64_t* offset) {
  if (!m || p < 0 || p >= (int)m->params.size()) return DPG_ERR_PARAMETER;
  const ParamInfo& pi = m->params[p];
  if (layer) *layer = pi.layer;
  if (slot) *slot = pi.slot;
  if (numel) *numel = pi.numel;
  if (offset) *offset = pi.offset;
  return DPG_OK;
}

dpg_status dpg_model_load_params(dpg_model* m, const float* host) {
  if (!m) return DPG_ERR_PARAMETER;
  return guard(m->ctx, [&] {
    DPG_CUDA(cudaSetDevice(m->ctx->device));
    DPG_CUDA(cudaMemcpyAsync(m->p_params, host, sizeof(float) * m->L, cudaMemcpyHostToDevice, m->ctx->stream));
    DPG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  });
}

dpg_status dpg_model_store_params(dpg_model* m, float* host) {
  if (!m) return DPG_ERR_PARAMETER;
  return guard(m->ctx, [&] {
    DPG_CUDA(cudaSetDevice(m->ctx->device));
    DPG_CUDA(cudaMemcpyAsync(host, m->p_params, sizeof(float) * m->L, cudaMemcpyDeviceToHost, m->ctx->stream));
    DPG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  });
}

dpg_status dpg_optimizer_create(dpg_model* m, const dpg_optimizer_config* cfg, dpg_optimizer** out) {
  if (!out || !m || !cfg) return DPG_ERR_PARAMETER;
  *out = nullptr;
  dpg_optimizer* o = new dpg_optimizer();
  const dpg_status st = guard(m->ctx, [&] {
    DPG_CUDA(cudaSetDevice(m->ctx->device));
    // DpOptimizerConfig::check (optimizer.hpp:28-33)
    if (cfg->noise_multiplier < 0.0) raise(DPG_ERR_PARAMETER, "noise multiplier must be >= 0");
    if (!(cfg->max_grad_norm > 0.0)) raise(DPG_ERR_PARAMETER, "max grad norm must be > 0");
    if (!(cfg->learning_rate > 0.0)) raise(DPG_ERR_PARAMETER, "learning rate must be > 0");
    if (!(cfg->expected_batch_size > 0.0)) raise(DPG_ERR_PARAMETER, "expected batch size must be > 0");
    if (cfg->clipped_sum_from_record && !cfg->materialise_grad_sample)
      raise(DPG_ERR_PARAMETER, "clipped_sum_from_record needs materialise_grad_sample");
    o->m = m;
    o->cfg = *cfg;
    const int64_t B = m->max_b, L = m->L;
    int64_t bias_numel = 0;
    for (auto& pi : m->params)
      if (pi.is_bias) bias_numel = std::max(bias_numel, pi.offset + pi.numel);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t rec = cfg->materialise_grad_sample ? sizeof(float) * (size_t)(B * L) : sizeof(float) * (size_t)(B * bias_numel);
    // summed / reduced: L clipped-sum elements + the multi-rank status lane (noise.cu)
    size_t total = al(sizeof(float) * (L + 1)) + al(sizeof(float) * L) + al(rec) + al(sizeof(double) * m->sq_rows * B) +
                   al(sizeof(double) * B) + al(sizeof(float) * B) + al(sizeof(int64_t)) + al(sizeof(uint64_t)) +
                   al(sizeof(float) * (L + 1)) + al(3 * 128) + al(sizeof(unsigned long long));
    DPG_CUDA(cudaMalloc(&o->arena, total));
    DPG_CUDA(cudaMemset(o->arena, 0, total));
    char* p = o->arena;
    auto take = [&](size_t bytes) {
      char* r = p;
      p += al(bytes);
      return r;
    };
    o->summed = reinterpret_cast<float*>(take(sizeof(float) * (L + 1)));
    o->grad = reinterpret_cast<float*>(take(sizeof(float) * L));
    float* r = reinterpret_cast<float*>(take(rec));
    if (cfg->materialise_grad_sample) o->record = r; else o->bias_scratch = r;
    o->slab = reinterpret_cast<double*>(take(sizeof(double) * m->sq_rows * B));
    o->norms = reinterpret_cast<double*>(take(sizeof(double) * B));
    o->scale = reinterpret_cast<float*>(take(sizeof(float) * B));
    o->num_clipped = reinterpret_cast<int64_t*>(take(sizeof(int64_t)));
    o->step_dev = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t)));
    o->reduced = reinterpret_cast<float*>(take(sizeof(float) * (L + 1)));
    o->xflags = reinterpret_cast<unsigned long long*>(take(3 * 128));
    o->step_tick = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long)));
  });
  if (st != DPG_OK) {
    if (o->arena) cudaFree(o->arena);
    delete o;
    return st;
  }
  *out = o;
  return DPG_OK;
}

void dpg_optimizer_destroy(dpg_optimizer* o) {
  if (!o) return;
  cudaSetDevice(o->m->ctx->device);
  cudaStreamSynchronize(o->m->ctx->stream);
  for (auto& g : o->graphs) cudaGraphExecDestroy(g.exec);
  for (auto e : o->ring_ev)
    if (e) cudaEventDestroy(e);
  if (o->step_ring) cudaFreeHost(o->step_ring);
  for (void* p : o->peer_maps) cudaIpcCloseMemHandle(p);
  if (o->arena) cudaFree(o->arena);
  delete o;
}

namespace {
struct PeerHandle {
  cudaIpcMemHandle_t arena;
  int64_t summed_off, flags_off, L;
};
static_assert(sizeof(PeerHandle) <= DPG_PEER_HANDLE_BYTES, "peer handle");
}  // namespace

dpg_status dpg_optimizer_peer_handle(dpg_optimizer* o, void* handle) {
  if (!o || !handle) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    DPG_CUDA(cudaSetDevice(o->m->ctx->device));
    PeerHandle h{};
    DPG_CUDA(cudaIpcGetMemHandle(&h.arena, o->arena));
    h.summed_off = reinterpret_cast<char*>(o->summed) - o->arena;
    h.flags_off = reinterpret_cast<char*>(o->xflags) - o->arena;
    h.L = o->m->L;
    std::memset(handle, 0, DPG_PEER_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof(h));
  });
}

dpg_status dpg_optimizer_set_peers(dpg_optimizer* o, int rank, int world, const void* handles) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    DPG_CUDA(cudaSetDevice(o->m->ctx->device));
    if (world < 1 || world > dpg::kMaxPeers || rank < 0 || rank >= world)
      raise(DPG_ERR_PARAMETER, "peer exchange: need 0 <= rank < world <= " + std::to_string(dpg::kMaxPeers));
    if (world > 1 && !handles) raise(DPG_ERR_PARAMETER, "peer exchange: handles must not be NULL");
    DPG_CUDA(cudaStreamSynchronize(o->m->ctx->stream));
    dpg::PeerSet ps;
    std::vector<void*> maps;
    if (world > 1) {
      ps.world = world;
      ps.rank = rank;
      for (int r = 0; r < world; ++r) {
        PeerHandle h;
        std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * DPG_PEER_HANDLE_BYTES, sizeof(h));
        if (h.L != o->m->L) raise(DPG_ERR_DIMENSION, "peer exchange: rank " + std::to_string(r) + " has " +
                                                         std::to_string(h.L) + " parameters, this rank " +
                                                         std::to_string(o->m->L));
        char* base = o->arena;
        if (r != rank) {
          void* p = nullptr;
          const cudaError_t e = cudaIpcOpenMemHandle(&p, h.arena, cudaIpcMemLazyEnablePeerAccess);
          if (e != cudaSuccess) {
            for (void* q : maps) cudaIpcCloseMemHandle(q);
            raise(DPG_ERR_CUDA, std::string("peer exchange: cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
          }
          maps.push_back(p);
          base = static_cast<char*>(p);
        }
        ps.summed[r] = reinterpret_cast<const float*>(base + h.summed_off);
        ps.flags[r] = reinterpret_cast<unsigned long long*>(base + h.flags_off);
      }
    }
    for (void* p : o->peer_maps) cudaIpcCloseMemHandle(p);
    o->peer_maps = maps;
    o->peers = ps;
    // captured steps bake the exchange in or out
    for (auto& g : o->graphs) cudaGraphExecDestroy(g.exec);
    o->graphs.clear();
  });
}

dpg_status dpg_forward_backward(dpg_optimizer* o, const float* x, const float* targets, int64_t b,
                                float* loss) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    DPG_CUDA(cudaSetDevice(o->m->ctx->device));
    if (b <= 0) raise(DPG_ERR_DIMENSION, "compute_grad_samples: batch must be non-empty");
    if (b > o->m->max_b)
      raise(DPG_ERR_DIMENSION, "batch " + std::to_string(b) + " exceeds the model's max_batch " +
                                   std::to_string(o->m->max_b));
    if (!x || !targets) raise(DPG_ERR_PARAMETER, "input and targets must not be NULL");
    check_set_grad_sample(o);
    forward_backward_impl(o, x, targets, b, loss);
    o->has_grad_sample = true;
    o->consumed = false;
    o->pending_b = b;
    o->pending_x = x;
  });
}

dpg_status dpg_virtual_step(dpg_optimizer* o) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    // optimizer.hpp:166-174
    if (!o->has_grad_sample || o->consumed)
      raise(DPG_ERR_LIFECYCLE, "virtual_step without a fresh grad_sample (run a backward first)");
    fold_impl(o, o->pending_b, o->pending_x);
    o->has_grad_sample = false;
    o->consumed = false;
  });
}

dpg_status dpg_step(dpg_optimizer* o) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] { step_impl(o, o->pending_x, false); });
}

dpg_status dpg_step_empty_batch(dpg_optimizer* o) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    // optimizer.hpp:197-213
    if (o->has_grad) raise(DPG_ERR_LIFECYCLE, "step called twice without zero_grad in between");
    if ((o->has_grad_sample && !o->consumed) || o->has_summed)
      raise(DPG_ERR_LIFECYCLE, "step_empty_batch with gradients pending");
    DPG_CUDA(cudaMemsetAsync(o->summed, 0, sizeof(float) * o->m->L, o->m->ctx->stream));
    o->has_summed = true;
    o->accumulated = 0;
    finish_impl(o, false);
  });
}

dpg_status dpg_zero_grad(dpg_optimizer* o) {
  if (!o) return DPG_ERR_PARAMETER;
  zero_grad_impl(o);
  return DPG_OK;
}

dpg_status dpg_set_noise_multiplier(dpg_optimizer* o, double sigma) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    if (sigma < 0.0) raise(DPG_ERR_PARAMETER, "noise multiplier must be >= 0");
    o->cfg.noise_multiplier = sigma;
    for (auto& g : o->graphs) cudaGraphExecDestroy(g.exec);
    o->graphs.clear();
  });
}

dpg_status dpg_set_expected_batch_size(dpg_optimizer* o, double e) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    if (!(e > 0.0)) raise(DPG_ERR_PARAMETER, "expected batch size must be > 0");
    o->cfg.expected_batch_size = e;
    for (auto& g : o->graphs) cudaGraphExecDestroy(g.exec);
    o->graphs.clear();
  });
}

dpg_status dpg_set_injected_noise(dpg_optimizer* o, const float* noise) {
  if (!o) return DPG_ERR_PARAMETER;
  o->injected = noise;
  for (auto& g : o->graphs) cudaGraphExecDestroy(g.exec);
  o->graphs.clear();
  return DPG_OK;
}

dpg_status dpg_last_clip_summary(dpg_optimizer* o, double* norms, double* scales,
                                 int64_t* num_clipped) {
  if (!o) return DPG_ERR_PARAMETER;
  return guard(o->m->ctx, [&] {
    dpg_ctx* ctx = o->m->ctx;
    surface(o->m);
    const int64_t b = o->last_b;
    if (norms && b) DPG_CUDA(cudaMemcpy(norms, o->norms, sizeof(double) * b, cudaMemcpyDeviceToHost));
    if (scales && b) {
      // scale_factors are doubles in the reference (C / max(N, C)); recompute from the norms
      std::vector<double> nrm(b);
      DPG_CUDA(cudaMemcpy(nrm.data(), o->norms, sizeof(double) * b, cudaMemcpyDeviceToHost));
      const double c = o->cfg.max_grad_norm;
      for (int64_t i = 0; i < b; ++i) scales[i] = c / std::max(nrm[i], c);
    }
    if (num_clipped) DPG_CUDA(cudaMemcpy(num_clipped, o->num_clipped, sizeof(int64_t), cudaMemcpyDeviceToHost));
    (void)ctx;
  });
}

// the pending batch's per-sample gradients of parameter p ([b, ...param], grad_sample.hpp:18-19) to
// the host; synchronous (GradSampleRecord export)
dpg_status dpg_grad_sample_export(const dpg_optimizer* o, int p, float* host, int64_t capacity) {
  return guard(o ? o->m->ctx : nullptr, [&] {
    if (!o) raise(DPG_ERR_PARAMETER, "null optimizer");
    if (p < 0 || p >= (int)o->m->params.size()) raise(DPG_ERR_PARAMETER, "parameter index out of range");
    if (!o->has_grad_sample) raise(DPG_ERR_LIFECYCLE, "no grad_sample: run forward_backward first");
    if (!o->cfg.materialise_grad_sample)
      raise(DPG_ERR_LIFECYCLE, "grad_sample was not materialised (materialise_grad_sample = 0)");
    const ParamInfo& pi = o->m->params[p];
    const int64_t n = o->pending_b * pi.numel;
    if (!host || capacity < n) raise(DPG_ERR_DIMENSION, "export buffer needs " + std::to_string(n) + " floats");
    DPG_CUDA(cudaSetDevice(o->m->ctx->device));
    DPG_CUDA(cudaStreamSynchronize(o->m->ctx->stream));
    DPG_CUDA(cudaMemcpy(host, o->record + o->pending_b * pi.offset, sizeof(float) * n, cudaMemcpyDeviceToHost));
  });
}

const float* dpg_grad_sample(const dpg_optimizer* o) {
  return (o && o->has_grad_sample && o->cfg.materialise_grad_sample) ? o->record : nullptr;
}
const float* dpg_summed_grad(const dpg_optimizer* o) { return (o && o->has_summed) ? o->summed : nullptr; }
const float* dpg_grad(const dpg_optimizer* o) { return (o && o->has_grad) ? o->grad : nullptr; }
int64_t dpg_accumulated_samples(const dpg_optimizer* o) { return o ? o->accumulated : 0; }

namespace {

// opt-in (DPG_PERSIST=1, read per call): measured slower than the multi-kernel step on the
// BASELINE small config (MNIST CNN b = 64: 0.227 vs 0.074 ms per step), see DESIGN.md §4c
bool persist_enabled() {
  const char* e = std::getenv("DPG_PERSIST");
  return e && e[0] == '1';
}

// Does a fresh logical batch of this model fit the persistent single-kernel step (persist.cu)?
// Small models and batches only: the kernel's phases are plain grid-stride loops, which win over
// the multi-kernel step only while launches, not work, bound it.
bool persist_ok(const dpg_optimizer* o, int64_t b) {
  const dpg_model* m = o->m;
  if (!persist_enabled() || !o->cfg.materialise_grad_sample || o->peers.world > 1 || m->ctx->comm ||
      m->ctx->profiling || m->out_width > 64 || b > 1024 || m->params.size() > (size_t)dpg::ps::kMaxParams)
    return false;
  int nl = 0;
  double macs = 0.0;
  for (const auto& lp : m->layers) {
    if (lp.kind == DPG_LAYER_RELU || lp.kind == DPG_LAYER_FLATTEN) continue;
    if (lp.kind == DPG_LAYER_LINEAR && lp.mid == 1) macs += (double)lp.out_numel * lp.d.in_features;
    else if (lp.kind == DPG_LAYER_CONV2D) macs += (double)lp.out_numel * lp.g.K();
    else return false;
    if (++nl > dpg::ps::kMaxLayers) return false;
  }
  if (macs * b > 4.0e7) return false;  // MNIST CNN b = 64: 1.7e7
  // a sample's input, activations and highways in shared memory
  int64_t floats = 0;
  for (const auto& lp : m->layers)
    if (lp.param0 >= 0) floats += (floats == 0 ? lp.in_numel : 0) + 2 * lp.out_numel;
  return 4 * floats <= 200 * 1024;
}

// the whole step (forward_backward + step of a fresh batch) as one cooperative launch
void persist_step(dpg_optimizer* o, const float* x, const float* targets, int64_t b, float* loss, bool graph_mode) {
  dpg_model* m = o->m;
  float* P = m->p_params;
  dpg::ps::Params p{};
  int li = 0;
  int64_t smem = 0;
  for (const auto& lp : m->layers) {
    if (lp.param0 < 0) continue;
    dpg::ps::PLayer& L = p.L[li++];
    L.conv = lp.kind == DPG_LAYER_CONV2D;
    L.in_relu = lp.in_relu ? 1 : 0;
    if (L.conv) {
      L.C = (int)lp.g.ic; L.H = (int)lp.g.h; L.W = (int)lp.g.w; L.O = (int)lp.g.oc; L.KH = (int)lp.g.kh;
      L.KW = (int)lp.g.kw; L.S = (int)lp.g.stride; L.PAD = (int)lp.g.pad; L.OH = (int)lp.g.oh; L.OW = (int)lp.g.ow;
    } else {
      L.C = (int)lp.d.in_features;
      L.O = (int)lp.d.out_features;
    }
    L.in_numel = lp.in_numel;
    L.out_numel = lp.out_numel;
    L.in = lp.in_buf < 0 ? x : nullptr;
    const ParamInfo& pw = m->params[lp.param0];
    L.w = P + pw.offset;
    L.bias = lp.nparams > 1 ? P + m->params[lp.param0 + 1].offset : nullptr;
    L.gw = o->record + b * pw.offset;
    L.gb = lp.nparams > 1 ? o->record + b * m->params[lp.param0 + 1].offset : nullptr;
    L.numel_w = pw.numel;
    L.pw = lp.param0;
    // shared memory of one sample: the input, then per layer its output and highway
    L.in_s = li == 1 ? 0 : p.L[li - 2].out_s;
    if (li == 1) smem = lp.in_numel;
    L.out_s = (int)smem;
    L.hw_s = (int)(smem + lp.out_numel);
    L.hw_prev_s = li == 1 ? -1 : p.L[li - 2].hw_s;
    smem += 2 * lp.out_numel;
  }
  smem *= 4;
  p.nl = li;
  p.b = b;
  p.out_relu = m->out_relu ? 1 : 0;
  p.targets = targets;
  p.loss = loss;
  p.np = (int)m->params.size();
  for (int q = 0; q < p.np; ++q) {
    p.rec[q] = o->record + b * m->params[q].offset;
    p.numel[q] = m->params[q].numel;
    p.off[q] = m->params[q].offset;
  }
  p.Ltot = m->L;
  p.c = o->cfg.max_grad_norm;
  p.part = o->slab;
  p.norms = o->norms;
  p.scale = o->scale;
  p.num_clipped = reinterpret_cast<long long*>(o->num_clipped);
  p.summed = o->summed;
  p.grad = o->grad;
  p.params = P;
  p.std_dev = o->cfg.noise_multiplier * o->cfg.max_grad_norm;
  p.inv_e = 1.0f / (float)o->cfg.expected_batch_size;
  p.lr = (float)o->cfg.learning_rate;
  p.seed = o->cfg.noise_seed;
  p.step = o->steps;
  p.step_ptr = graph_mode ? o->step_dev : nullptr;
  p.injected = o->injected;
  p.err = m->ctx->dev_err;
  p.bar = m->persist_bar;
  dpg::ProfScope ps(m->ctx, "persist.step", 0.0, 0.0);
  dpg::launch_persist_step(m->ctx, p, (int)smem);
}

}  // namespace

dpg_status dpg_train_step(dpg_optimizer* o, const float* x, const float* targets, int64_t b,
                          float* loss, int use_graph) {
  if (!o) return DPG_ERR_PARAMETER;
  dpg_model* m = o->m;
  dpg_ctx* ctx = m->ctx;
  return guard(ctx, [&] {
    DPG_CUDA(cudaSetDevice(ctx->device));
    if (b <= 0) raise(DPG_ERR_DIMENSION, "compute_grad_samples: batch must be non-empty");
    if (b > m->max_b) raise(DPG_ERR_DIMENSION, "batch exceeds the model's max_batch");
    if (!x || !targets) raise(DPG_ERR_PARAMETER, "input and targets must not be NULL");
    // a train step opens a fresh logical batch: zero_grad, forward_backward, step
    zero_grad_impl(o);
    auto mark_done = [&] {
      o->has_grad_sample = true;
      o->consumed = true;
      o->has_summed = true;
      o->has_grad = true;
      o->accumulated = b;
      o->last_b = b;
      o->pending_b = b;
      o->pending_x = x;
    };
    const bool persist = persist_ok(o, b);
    if (!use_graph) {
      if (persist) {
        persist_step(o, x, targets, b, loss, false);
        mark_done();
        ++o->steps;
        o->dev_step_known = false;
        return;
      }
      forward_backward_impl(o, x, targets, b, loss);
      o->has_grad_sample = true;
      o->pending_b = b;
      o->pending_x = x;
      step_impl(o, x, false);
      return;
    }
    if (o->graph_comm_gen != ctx->comm_gen) {
      // the communicator changed (dpg_ctx_init_comm): graphs captured with the old one (or with
      // none) would all-reduce on a destroyed communicator or not at all
      DPG_CUDA(cudaStreamSynchronize(ctx->stream));
      for (auto& g : o->graphs) cudaGraphExecDestroy(g.exec);
      o->graphs.clear();
      o->graph_comm_gen = ctx->comm_gen;
    }
    dpg_optimizer::Graph* hit = nullptr;
    for (auto& g : o->graphs)
      if (g.b == b && g.x == x && g.y == targets && g.loss == loss) hit = &g;
    if (!hit) {
      cudaGraph_t graph;
      const int64_t before = ctx->launches;
      ctx->capturing = true;
      DPG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      if (ctx->timeline) DPG_CUDA(cudaEventRecordWithFlags(ctx->tl_start, ctx->stream, cudaEventRecordExternal));
      try {
        if (persist) {
          persist_step(o, x, targets, b, loss, true);
        } else {
          forward_backward_impl(o, x, targets, b, loss);
          o->has_grad_sample = true;
          o->pending_b = b;
          o->pending_x = x;
          step_impl(o, x, true);
        }
      } catch (...) {
        cudaStreamEndCapture(ctx->stream, &graph);
        ctx->capturing = false;
        zero_grad_impl(o);
        throw;
      }
      DPG_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
      ctx->capturing = false;
      const int64_t kernels = ctx->launches - before;
      ctx->launches = before;
      if (o->graphs.size() >= dpg_optimizer::kMaxGraphs) {
        auto lru = std::min_element(o->graphs.begin(), o->graphs.end(),
                                    [](const auto& a, const auto& c) { return a.last_use < c.last_use; });
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(lru->exec, graph, &info) == cudaSuccess) {
          *lru = {b, x, targets, loss, lru->exec, kernels, 0};
          hit = &*lru;
        } else {
          (void)cudaGetLastError();  // topology changed (e.g. another split-K choice): rebuild
          DPG_CUDA(cudaGraphExecDestroy(lru->exec));
          o->graphs.erase(lru);
        }
      }
      if (!hit) {
        cudaGraphExec_t exec;
        DPG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        o->graphs.push_back({b, x, targets, loss, exec, kernels, 0});
        hit = &o->graphs.back();
      }
      DPG_CUDA(cudaGraphDestroy(graph));
    }
    hit->last_use = ++o->graph_clock;
    if (!o->step_ring) {
      DPG_CUDA(cudaHostAlloc(&o->step_ring, sizeof(uint64_t) * dpg_optimizer::kStepRing, cudaHostAllocDefault));
      for (auto& e : o->ring_ev) DPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (!o->dev_step_known || o->dev_step_next != o->steps) {
      const int slot = (int)(o->steps % dpg_optimizer::kStepRing);
      if (o->ring_used[slot]) DPG_CUDA(cudaEventSynchronize(o->ring_ev[slot]));
      o->step_ring[slot] = o->steps;
      DPG_CUDA(cudaMemcpyAsync(o->step_dev, &o->step_ring[slot], sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
      DPG_CUDA(cudaEventRecord(o->ring_ev[slot], ctx->stream));
      o->ring_used[slot] = true;
    }
    DPG_CUDA(cudaGraphLaunch(hit->exec, ctx->stream));
    ctx->launches += hit->kernels;
    ++o->steps;
    o->dev_step_known = true;  // the replay's update kernel wrote steps + 1 ... i.e. the new o->steps
    o->dev_step_next = o->steps;
    mark_done();
  });
}

dpg_status dpg_train_step_host(dpg_optimizer* o, const float* x_host, const float* targets_host,
                               int64_t b, float* loss_host) {
  if (!o) return DPG_ERR_PARAMETER;
  dpg_model* m = o->m;
  dpg_ctx* ctx = m->ctx;
  const dpg_status st = guard(ctx, [&] {
    DPG_CUDA(cudaSetDevice(ctx->device));
    if (b <= 0) raise(DPG_ERR_DIMENSION, "compute_grad_samples: batch must be non-empty");
    if (b > m->max_b) raise(DPG_ERR_DIMENSION, "batch exceeds the model's max_batch");
    DPG_CUDA(cudaMemcpyAsync(m->x_stage, x_host, sizeof(float) * b * m->in_numel, cudaMemcpyHostToDevice, ctx->stream));
    DPG_CUDA(cudaMemcpyAsync(m->y_stage, targets_host, sizeof(float) * b, cudaMemcpyHostToDevice, ctx->stream));
  });
  if (st != DPG_OK) return st;
  const dpg_status st2 = dpg_train_step(o, m->x_stage, m->y_stage, b, m->loss, 1);
  if (st2 != DPG_OK) return st2;
  return guard(ctx, [&] {
    if (loss_host)
      DPG_CUDA(cudaMemcpyAsync(loss_host, m->loss, sizeof(float) * b, cudaMemcpyDeviceToHost, ctx->stream));
    try {
      surface(m);
    } catch (...) {
      zero_grad_impl(o);
      throw;
    }
  });
}

// Pipelined host path: the H2D of call k goes to staging slot k % 2 on the model's copy stream
// (after the step that last read that slot), the step waits for it on the compute stream, and
// the loss D2H follows the step. Nothing blocks the host, so the copies of step k + 1 overlap
// the kernels of step k.
dpg_status dpg_train_step_host_async(dpg_optimizer* o, const float* x_host, const float* targets_host,
                                     int64_t b, float* loss_host) {
  if (!o) return DPG_ERR_PARAMETER;
  dpg_model* m = o->m;
  dpg_ctx* ctx = m->ctx;
  int slot = 0;
  const dpg_status st = guard(ctx, [&] {
    DPG_CUDA(cudaSetDevice(ctx->device));
    if (b <= 0) raise(DPG_ERR_DIMENSION, "compute_grad_samples: batch must be non-empty");
    if (b > m->max_b) raise(DPG_ERR_DIMENSION, "batch exceeds the model's max_batch");
    if (!x_host || !targets_host) raise(DPG_ERR_PARAMETER, "input and targets must not be NULL");
    if (!m->copy_stream) {
      DPG_CUDA(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
      DPG_CUDA(cudaStreamCreateWithFlags(&m->read_stream, cudaStreamNonBlocking));
      ctx->extra_streams.push_back(m->read_stream);
      for (int q = 0; q < 2; ++q) {
        DPG_CUDA(cudaEventCreateWithFlags(&m->copied[q], cudaEventDisableTiming));
        DPG_CUDA(cudaEventCreateWithFlags(&m->consumed[q], cudaEventDisableTiming));
        DPG_CUDA(cudaEventCreateWithFlags(&m->loss_read[q], cudaEventDisableTiming));
      }
    }
    slot = (int)(m->async_calls & 1);
    if (m->async_calls >= 2) {
      DPG_CUDA(cudaStreamWaitEvent(m->copy_stream, m->consumed[slot], 0));
      DPG_CUDA(cudaStreamWaitEvent(ctx->stream, m->loss_read[slot], 0));  // slot's loss copied out
    }
    DPG_CUDA(cudaMemcpyAsync(m->xs[slot], x_host, sizeof(float) * b * m->in_numel, cudaMemcpyHostToDevice, m->copy_stream));
    DPG_CUDA(cudaMemcpyAsync(m->ys[slot], targets_host, sizeof(float) * b, cudaMemcpyHostToDevice, m->copy_stream));
    DPG_CUDA(cudaEventRecord(m->copied[slot], m->copy_stream));
    DPG_CUDA(cudaStreamWaitEvent(ctx->stream, m->copied[slot], 0));
    ++m->async_calls;
  });
  if (st != DPG_OK) return st;
  const dpg_status st2 = dpg_train_step(o, m->xs[slot], m->ys[slot], b, m->losses[slot], 1);
  if (st2 != DPG_OK) return st2;
  return guard(ctx, [&] {
    DPG_CUDA(cudaEventRecord(m->consumed[slot], ctx->stream));
    // the loss read-back rides on the copy stream, off the compute stream's step-to-step path
    DPG_CUDA(cudaStreamWaitEvent(m->read_stream, m->consumed[slot], 0));
    if (loss_host)
      DPG_CUDA(cudaMemcpyAsync(loss_host, m->losses[slot], sizeof(float) * b, cudaMemcpyDeviceToHost,
                               m->read_stream));
    DPG_CUDA(cudaEventRecord(m->loss_read[slot], m->read_stream));
  });
}

}  // extern "C"
