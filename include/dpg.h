/*
 * dpg.h — C ABI of the B200-native DP-SGD step (libdpg.so).
 *
 * The drop-in boundary for the hot path of the reference C++ library `dpgrad`
 * (/root/reference/proj/core): per-sample gradients, per-sample norm, clip + clipped sum,
 * noise + SGD update. Plain C: pointers, sizes, status codes; no C++ or torch types.
 *
 * Every entry point names the reference interface it replaces. Two layers:
 *
 *   1. Operator ABI (device pointers, asynchronous on the context's stream): one call per
 *      reference operator — the per-layer GradSampleRule bodies (grad_sample.hpp:53-150),
 *      clip_and_sum (optimizer.hpp:62-116), add_noise + finish_step (optimizer.hpp:120-133,
 *      256-271). This is what a GradSampleRule adapter registered with
 *      GradSamplerRegistry::register_rule(kind, rule, override_existing=true)
 *      (grad_sample.hpp:159-167) calls; see INTEGRATION.md.
 *
 *   2. Engine ABI: a device-resident ModelGraph + GradSampleModule + DpOptimizer
 *      (layers.hpp:227-245, optimizer.hpp:138-278, 359-381) that runs the whole step on the
 *      GPU with the reference's lifecycle (set_grad_sample -> virtual_step* -> step ->
 *      zero_grad) and error contract, plus one NCCL all-reduce of the clipped sum when the
 *      context has a communicator.
 *
 * Errors: no exceptions cross the ABI. Each call returns dpg_status whose values map 1:1 onto
 * the reference exception classes (errors.hpp:12-72); dpg_last_error() holds the message with
 * the same fields the reference prints (layer, parameter name, sample). Errors detected on the
 * device (non-finite per-sample gradient, out-of-range index or target) are recorded in a
 * device status word and returned by the next synchronising call (dpg_ctx_sync, or any engine
 * call that reads results back); the device stages after the faulting one become no-ops, so the
 * parameters stay untouched exactly as when the reference throws out of clip_and_sum.
 *
 * Layouts are the reference's: row-major, per-sample tensors [b, ...param shape]
 * (grad_sample.hpp:18-19), parameters in (layer, slot) order weight, bias / table
 * (layers.hpp:933-969), conv inputs NCHW, linear inputs [b, mid..., features].
 */
#ifndef DPG_H
#define DPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPG_API __attribute__((visibility("default")))
#define DPG_ABI_VERSION 2

/* errors.hpp:12-72 */
typedef enum dpg_status {
  DPG_OK = 0,
  DPG_ERR_DIMENSION = 1, /* DimensionError  (errors.hpp:20-23) */
  DPG_ERR_PARAMETER = 2, /* ParameterError  (errors.hpp:26-29) */
  DPG_ERR_LIFECYCLE = 3, /* LifecycleError  (errors.hpp:33-36) */
  DPG_ERR_REGISTRY = 4,  /* RegistryError   (errors.hpp:39-42) */
  DPG_ERR_NUMERIC = 5,   /* NumericError    (errors.hpp:45-48) */
  DPG_ERR_CUDA = 6,
  DPG_ERR_NCCL = 7,
  DPG_ERR_INTERNAL = 8,
} dpg_status;

/* LayerKind (layers.hpp:19-30) */
typedef enum dpg_layer_kind {
  DPG_LAYER_LINEAR = 0,
  DPG_LAYER_EMBEDDING = 1,
  DPG_LAYER_CONV2D = 2,
  DPG_LAYER_LAYER_NORM = 3, /* over the trailing norm_size features (1-D normalized shape) */
  DPG_LAYER_GROUP_NORM = 4, /* groups over norm_size channels of [batch, C, ...] */
  DPG_LAYER_RELU = 5,
  DPG_LAYER_FLATTEN = 6,
} dpg_layer_kind;

/* LayerDescriptor (layers.hpp:69-194), hot-path fields; see configs.py CLayerDesc. */
typedef struct dpg_layer_desc {
  int32_t kind;
  int32_t has_bias;
  int64_t in_features, out_features; /* linear */
  int64_t vocab_size, embedding_dim; /* embedding */
  int64_t in_channels, out_channels, kernel_h, kernel_w, stride, padding; /* conv2d */
  int64_t norm_size, groups; /* layer_norm: normalized numel; group_norm: channels, groups */
  double eps;                /* layer_norm / group_norm (layers.hpp:128-150, default 1e-5) */
} dpg_layer_desc;

/* Conv2dSpec (layers.hpp:58-65); groups = dilation = 1 as in the reference. */
typedef struct dpg_conv2d_spec {
  int64_t in_channels, out_channels, kernel_h, kernel_w, stride, padding;
} dpg_conv2d_spec;

typedef struct dpg_ctx dpg_ctx;

/* ======================================================================================
 * Context
 * ====================================================================================== */

DPG_API int dpg_abi_version(void);

/* One context per (host thread, GPU). `stream` is a cudaStream_t (NULL: the context creates
 * its own non-blocking stream). Not thread-safe (single-owner, like RngStream, rng.hpp:16). */
DPG_API dpg_status dpg_ctx_create(int device, void* stream, dpg_ctx** out);
DPG_API void dpg_ctx_destroy(dpg_ctx* ctx);
DPG_API void* dpg_ctx_stream(const dpg_ctx* ctx);

/* Message of the last failure (per context; per thread when ctx is NULL). */
DPG_API const char* dpg_last_error(const dpg_ctx* ctx);

/* Synchronise the stream and surface any error recorded on the device since the last check. */
DPG_API dpg_status dpg_ctx_sync(dpg_ctx* ctx);

/* Number of kernels this context has launched (evidence for bench.py's gpu_launches). */
DPG_API int64_t dpg_ctx_kernel_launches(const dpg_ctx* ctx);

/* Stage profiling of eager (non-graph) launches: CUDA events on the context stream around each
 * stage. dpg_ctx_profile_read synchronises and returns one line per stage:
 *   "<stage> <total_ms> <count> <algorithmic_bytes_total> <algorithmic_flops_total>\n"
 * (the string stays valid until the next call). Enabling clears the aggregate. */
DPG_API dpg_status dpg_ctx_set_profiling(dpg_ctx* ctx, int on);
DPG_API const char* dpg_ctx_profile_read(dpg_ctx* ctx);

/* Graph timeline: while on, the stage scopes of a step captured by dpg_train_step become CUDA
 * event-record nodes on the stream (main or branch) that runs each stage, so a replay shows the
 * step's real overlap. Turning it on (or off) clears the records; steps captured before keep no
 * records. dpg_ctx_timeline_read synchronises the device and returns, for the last replay, one
 * line per stage scope in capture order:
 *   "<stage> <start_ms_from_graph_start> <duration_ms> <kernels>\n"
 * The record nodes split programmatic-dependent launch edges at stage boundaries, so the step
 * runs slightly slower than without them (a diagnostic, not a bench number). */
DPG_API dpg_status dpg_ctx_set_timeline(dpg_ctx* ctx, int on);
DPG_API const char* dpg_ctx_timeline_read(dpg_ctx* ctx);

/* NCCL: one communicator per context for the sample-sharded step.
 * dpg_nccl_unique_id fills 128 bytes on rank 0; every rank then calls dpg_ctx_init_comm. */
DPG_API dpg_status dpg_nccl_unique_id(unsigned char id[128]);
DPG_API dpg_status dpg_ctx_init_comm(dpg_ctx* ctx, int nranks, int rank, const unsigned char id[128]);
/* In-place sum over ranks of n floats on the context's stream (the clipped-sum exchange). */
DPG_API dpg_status dpg_allreduce_sum(dpg_ctx* ctx, float* buf, int64_t n);

/* ======================================================================================
 * Operator ABI — device pointers, asynchronous on the context stream.
 *
 * Norm partials: every grad-sample operator can also emit ||g_n||^2 of each parameter it
 * produces, accumulated in double from the fp32 values it stores (optimizer.hpp:72-86), as
 * sq_* [b]. Passing NULL skips that output; passing NULL for the gradient output (gw / g)
 * computes the norm without materialising the per-sample gradient.
 * ====================================================================================== */

/* per_sample_rule_linear (grad_sample.hpp:53-59) + registry "linear" (grad_sample.hpp:188-201):
 *   gw[n,o,i] = sum_t highway[n,t,o] * acts[n,t,i]   (batched_outer, tensor.hpp:303-338)
 *   gb[n,o]   = sum_t highway[n,t,o]                 (sum_middle, tensor.hpp:188-207)
 * acts [b, mid, d], highway [b, mid, r], gw [b, r, d], gb [b, r] (NULL: no bias). */
DPG_API dpg_status dpg_grad_sample_linear(dpg_ctx* ctx, const float* acts, const float* highway,
                                          int64_t b, int64_t mid, int64_t d, int64_t r, float* gw,
                                          float* gb, double* sq_w, double* sq_b);

/* per_sample_rule_conv2d (grad_sample.hpp:135-150): implicit im2col (layers.hpp:290-324), no
 * unfolded tensor in memory. x [b, ic, h, w], highway [b, oc, oh, ow],
 * gw [b, oc, ic, kh, kw], gb [b, oc] (NULL: no bias). */
DPG_API dpg_status dpg_grad_sample_conv2d(dpg_ctx* ctx, const float* x, const float* highway,
                                          int64_t b, int64_t h, int64_t w,
                                          const dpg_conv2d_spec* spec, float* gw, float* gb,
                                          double* sq_w, double* sq_b);

/* per_sample_rule_embedding (grad_sample.hpp:64-82): out[n, idx[n,s], :] += highway[n,s,:],
 * duplicates summed in ascending s. idx [b, t] holds token ids as float, as the reference
 * stores them (must be integral and < vocab, layers.hpp:368-376 -> DPG_ERR_PARAMETER).
 * g [b, vocab, dim] dense (NULL: sparse mode, norms only). */
DPG_API dpg_status dpg_grad_sample_embedding(dpg_ctx* ctx, const float* idx, const float* highway,
                                             int64_t b, int64_t t, int64_t vocab, int64_t dim,
                                             float* g, double* sq);

/* per_sample_rule_layer_norm (grad_sample.hpp:87-108), registry "layer_norm" (:216-220):
 *   ggamma[n,j] = sum_p highway[n,p,j] * normalized[n,p,j],  gbeta[n,j] = sum_p highway[n,p,j]
 * normalized / highway [b, positions, m] (normalized = the forward cache's xhat); fp32 sums in
 * ascending p as the reference (bit-identical). Either output may be NULL. */
DPG_API dpg_status dpg_grad_sample_layer_norm(dpg_ctx* ctx, const float* normalized, const float* highway,
                                              int64_t b, int64_t positions, int64_t m, float* ggamma,
                                              float* gbeta, double* sq_gamma, double* sq_beta);
/* per_sample_rule_group_norm (grad_sample.hpp:110-131), registry "group_norm" (:221-225):
 *   ggamma[n,c] = sum_s highway[n,c,s] * normalized[n,c,s],  gbeta[n,c] = sum_s highway[n,c,s]
 * normalized / highway [b, channels, spatial]. */
DPG_API dpg_status dpg_grad_sample_group_norm(dpg_ctx* ctx, const float* normalized, const float* highway,
                                              int64_t b, int64_t channels, int64_t spatial, float* ggamma,
                                              float* gbeta, double* sq_gamma, double* sq_beta);

/* clip_and_sum factors (optimizer.hpp:67-98): N_n = sqrt(sum_p sq[p, n]) summed in parameter
 * order; scale_n = (float)(C / max(N_n, C)); num_clipped = #{N_n > C}. A non-finite sq[p, n]
 * raises NumericError for the first (p, n) in the reference's scan order (p = index in (layer,
 * slot) order). sq [nparams, b] double; norms [b] double; scale [b] float; num_clipped: one
 * device int64 (nullable). Errors: C <= 0 or b == 0 -> DPG_ERR_PARAMETER (optimizer.hpp:64-65). */
DPG_API dpg_status dpg_clip_factors(dpg_ctx* ctx, const double* sq, int nparams, int64_t b,
                                    double c, double* norms, float* scale, int64_t* num_clipped);

/* Clipped sums without re-reading the per-sample gradients: (scale ⊙ B)^T A per layer
 * (clip_and_sum pass 2, optimizer.hpp:99-114, reassociated). accumulate != 0 adds into the
 * outputs (fold_pending across virtual steps, optimizer.hpp:240-254). */
DPG_API dpg_status dpg_clipped_sum_linear(dpg_ctx* ctx, const float* acts, const float* highway,
                                          const float* scale, int64_t b, int64_t mid, int64_t d,
                                          int64_t r, float* sw, float* sb, int accumulate);
DPG_API dpg_status dpg_clipped_sum_conv2d(dpg_ctx* ctx, const float* x, const float* highway,
                                          const float* scale, int64_t b, int64_t h, int64_t w,
                                          const dpg_conv2d_spec* spec, float* sw, float* sb,
                                          int accumulate);
/* Embedding: summed[v, :] = sum_n scale_n * (sum_{s: idx[n,s]=v} highway[n,s,:]) in ascending n
 * and s — the reference's association order, so it is bit-exact with clip_and_sum. */
DPG_API dpg_status dpg_clipped_sum_embedding(dpg_ctx* ctx, const float* idx, const float* highway,
                                             const float* scale, int64_t b, int64_t t,
                                             int64_t vocab, int64_t dim, float* summed,
                                             int accumulate);

/* clip_and_sum on materialised per-sample gradients, exact reference semantics and order
 * (optimizer.hpp:62-116) for any parameter (custom layers). g[p] / summed[p] are device
 * pointers passed in host arrays; numel[p] = per-sample element count. */
DPG_API dpg_status dpg_clip_and_sum_materialised(dpg_ctx* ctx, const float* const* g,
                                                 const int64_t* numel, int nparams, int64_t b,
                                                 double c, float* const* summed, double* norms,
                                                 float* scale, int64_t* num_clipped,
                                                 int accumulate);

/* Workspace: the operators above take scratch (norm partials, split-K partials, sort keys)
 * from one per-context device arena that grows on first use. To keep every hot call
 * allocation-free, query the largest size the caller will use and reserve it
 * once. A query returns 0 for invalid extents (the call itself reports the error). */
DPG_API size_t dpg_grad_sample_linear_workspace_size(int64_t b, int64_t mid, int64_t d, int64_t r);
DPG_API size_t dpg_grad_sample_conv2d_workspace_size(int64_t b, int64_t h, int64_t w,
                                                     const dpg_conv2d_spec* spec);
DPG_API size_t dpg_grad_sample_embedding_workspace_size(int64_t b, int64_t t, int64_t vocab, int64_t dim);
DPG_API size_t dpg_clipped_sum_linear_workspace_size(int64_t b, int64_t mid, int64_t d, int64_t r);
DPG_API size_t dpg_clipped_sum_conv2d_workspace_size(int64_t b, int64_t h, int64_t w,
                                                     const dpg_conv2d_spec* spec);
DPG_API size_t dpg_clipped_sum_embedding_workspace_size(int64_t b, int64_t t, int64_t vocab, int64_t dim);
DPG_API dpg_status dpg_ctx_reserve_workspace(dpg_ctx* ctx, size_t bytes);

/* add_noise + finish_step (optimizer.hpp:120-133, 256-271), fused, over n flat elements:
 *   noised = summed + (float)(N(0,1) * sigma * C)      sigma == 0: no noise
 *   grad   = noised * (1.0f / (float)E)                 (scale(), tensor.hpp:155-159)
 *   params = params - grad * (float)lr                  (two fp32 roundings, no FMA)
 * N(0,1) comes from counter-based Philox4x32-10 keyed by `seed`, counter (step, element pair)
 * + Box-Muller in double, so every rank draws the same noise without communication.
 * injected_noise (nullable) replaces the draws with a caller tensor (bit-parity with the
 * reference's mt19937_64 stream). grad (nullable) receives the averaged noisy gradient. */
DPG_API dpg_status dpg_noise_update(dpg_ctx* ctx, float* params, const float* summed, float* grad,
                                    int64_t n, double sigma, double c, double expected_batch,
                                    double lr, uint64_t seed, uint64_t step,
                                    const float* injected_noise);

/* The noise alone: out[i] = (float)(N(0,1) * std) from the same Philox stream (for tests). */
DPG_API dpg_status dpg_gaussian(dpg_ctx* ctx, float* out, int64_t n, double std_dev, uint64_t seed,
                                uint64_t step);

/* ======================================================================================
 * Engine ABI — device-resident ModelGraph + GradSampleModule + DpOptimizer.
 * ====================================================================================== */

typedef struct dpg_model dpg_model;
typedef struct dpg_optimizer dpg_optimizer;

/* build_model's graph (layers.hpp:926-973) on the device; parameters zero until loaded.
 * in_shape is the per-sample input shape (without the batch); max_batch bounds b for the
 * arenas, which are allocated once here (no allocation on the step path). */
DPG_API dpg_status dpg_model_create(dpg_ctx* ctx, const dpg_layer_desc* layers, int nlayers,
                                    const int64_t* in_shape, int in_rank, int64_t max_batch,
                                    dpg_model** out);
DPG_API void dpg_model_destroy(dpg_model* model);
/* ModelGraph::parameter_count (layers.hpp:231-237) */
DPG_API int64_t dpg_model_parameter_count(const dpg_model* model);
DPG_API int dpg_model_num_param_tensors(const dpg_model* model);
DPG_API dpg_status dpg_model_param_info(const dpg_model* model, int p, int* layer, int* slot,
                                        int64_t* numel, int64_t* offset);
/* Flat device parameter vector [L] in (layer, slot) order (writable). */
DPG_API float* dpg_model_params(dpg_model* model);
DPG_API dpg_status dpg_model_load_params(dpg_model* model, const float* host);
DPG_API dpg_status dpg_model_store_params(dpg_model* model, float* host);
/* Per-class logits width of the model output. */
DPG_API int64_t dpg_model_output_width(const dpg_model* model);

/* DpOptimizerConfig (optimizer.hpp:21-34) + the device noise seed. */
typedef struct dpg_optimizer_config {
  double noise_multiplier;    /* sigma */
  double max_grad_norm;       /* C */
  double learning_rate;
  double expected_batch_size; /* averaging denominator E (global, across ranks) */
  uint64_t noise_seed;        /* Philox key; identical on every rank */
  int32_t materialise_grad_sample; /* 1: keep the GradSampleRecord readable until zero_grad */
  int32_t clipped_sum_from_record; /* 1: clip_and_sum reads the record (reference pass 2);
                                      0: (scale ⊙ B)^T A without re-reading it (default) */
} dpg_optimizer_config;

DPG_API dpg_status dpg_optimizer_create(dpg_model* model, const dpg_optimizer_config* cfg,
                                        dpg_optimizer** out);
DPG_API void dpg_optimizer_destroy(dpg_optimizer* opt);

/* The clipped-sum exchange over peer memory instead of NCCL: every
 * rank maps the other ranks' optimizer state (CUDA IPC; NVLink P2P between GPUs) and step()
 * sums the W clipped sums straight from peer memory inside the noise + update kernel, in rank
 * order (identical on every rank), with device-side flags ordering the ranks — no all-reduce
 * launch, no host synchronisation. After step(), the summed buffer holds the all-rank sum, as
 * with dpg_allreduce_sum. Replaces ncclAllReduce (the reference's W = 1 analogue is the
 * virtual-step fold, optimizer.hpp:240-254).
 *   dpg_optimizer_peer_handle  writes this rank's DPG_PEER_HANDLE_BYTES-byte handle;
 *   dpg_optimizer_set_peers    takes all W handles (rank order, this rank's included); W = 1
 *                              turns the exchange off. Every rank must then call step() the
 *                              same number of times (a rank waits for its peers' clipped sums). */
#define DPG_PEER_HANDLE_BYTES 128
DPG_API dpg_status dpg_optimizer_peer_handle(dpg_optimizer* opt, void* handle);
DPG_API dpg_status dpg_optimizer_set_peers(dpg_optimizer* opt, int rank, int world, const void* handles);

/* GradSampleModule::forward_backward (optimizer.hpp:369-372) -> compute_grad_samples
 * (grad_sample.hpp:328-343) followed by DpOptimizer::set_grad_sample (optimizer.hpp:147-161):
 * one forward, softmax cross-entropy (layers.hpp:894-919), one backward walk with the device
 * rules, norm partials fused into the rule epilogues. x [b, in_shape] and targets [b] (class
 * ids as float, layers.hpp:905) are device pointers; loss [b] (nullable) receives the
 * per-sample loss. Lifecycle errors as set_grad_sample. */
DPG_API dpg_status dpg_forward_backward(dpg_optimizer* opt, const float* x, const float* targets,
                                        int64_t b, float* loss);
/* DpOptimizer::virtual_step / step / step_empty_batch / zero_grad (optimizer.hpp:166-222). With
 * a communicator on the context, step() all-reduces the clipped sum before the noise. */
DPG_API dpg_status dpg_virtual_step(dpg_optimizer* opt);
DPG_API dpg_status dpg_step(dpg_optimizer* opt);
DPG_API dpg_status dpg_step_empty_batch(dpg_optimizer* opt);
DPG_API dpg_status dpg_zero_grad(dpg_optimizer* opt);
DPG_API dpg_status dpg_set_noise_multiplier(dpg_optimizer* opt, double sigma);
DPG_API dpg_status dpg_set_expected_batch_size(dpg_optimizer* opt, double e);
/* Replace the Philox draws of the following steps by a device noise tensor [L] (NULL: Philox). */
DPG_API dpg_status dpg_set_injected_noise(dpg_optimizer* opt, const float* noise);

/* last_clip_summary (optimizer.hpp:225): synchronises; host arrays [b] (nullable). */
DPG_API dpg_status dpg_last_clip_summary(dpg_optimizer* opt, double* norms, double* scales,
                                         int64_t* num_clipped);
/* GradientState views (optimizer.hpp:47-57); NULL when the stage is absent. Device pointers.
 * grad_sample: flat record, parameter p occupies [b * offset_p, b * (offset_p + numel_p)). */
DPG_API const float* dpg_grad_sample(const dpg_optimizer* opt);
DPG_API const float* dpg_summed_grad(const dpg_optimizer* opt);
DPG_API const float* dpg_grad(const dpg_optimizer* opt);
DPG_API int64_t dpg_accumulated_samples(const dpg_optimizer* opt);

/* One whole DP-SGD step with HOST buffers (the end-to-end path): H2D of x and targets,
 * forward_backward, step, D2H of the per-sample loss [b] (nullable), zero_grad. Synchronous;
 * returns any device-detected error. */
DPG_API dpg_status dpg_train_step_host(dpg_optimizer* opt, const float* x_host,
                                       const float* targets_host, int64_t b, float* loss_host);
/* Pipelined variant of dpg_train_step_host for training loops: enqueues the H2D of x and
 * targets (into one of two device staging slots, on a copy stream), the step and the D2H of the
 * per-sample loss, and returns without waiting, so the copies of the next call overlap this
 * step's kernels. Host buffers must stay valid (pinned for overlap) until dpg_ctx_sync, which
 * also surfaces device-detected errors. Same semantics per step as dpg_train_step_host. */
DPG_API dpg_status dpg_train_step_host_async(dpg_optimizer* opt, const float* x_host,
                                             const float* targets_host, int64_t b, float* loss_host);
/* The same step on device buffers, asynchronous; replayed from a CUDA graph captured on the
 * first call for each batch size (set use_graph = 0 to launch eagerly). */
DPG_API dpg_status dpg_train_step(dpg_optimizer* opt, const float* x, const float* targets,
                                  int64_t b, float* loss, int use_graph);

/* ======================================================================================
 * Privacy bookkeeping (host side).
 *
 * NoiseSchedule (reference optimizer.hpp:280-358): sigma per epoch. dpg_noise_schedule_init
 * validates like the reference factories (constant / exponential / step / custom; the custom table
 * is borrowed, not copied); dpg_schedule_noise evaluates epoch, stores it in `current` and, when
 * opt is non-NULL, applies it (dpg_set_noise_multiplier). */
enum { DPG_SCHEDULE_CONSTANT = 0, DPG_SCHEDULE_EXPONENTIAL = 1, DPG_SCHEDULE_STEP = 2, DPG_SCHEDULE_CUSTOM = 3 };
typedef struct dpg_noise_schedule {
  int kind;
  double initial_sigma;
  double gamma;   /* exponential: sigma0 * gamma^epoch */
  double factor;  /* step: sigma0 * factor^(epoch / period) */
  uint64_t period;
  const double* table; /* custom: per-epoch values, the last persists */
  int64_t table_len;
  double current;
} dpg_noise_schedule;
DPG_API dpg_status dpg_noise_schedule_init(dpg_noise_schedule* s, int kind, double sigma0, double gamma,
                                           double factor, uint64_t period, const double* table,
                                           int64_t table_len);
DPG_API double dpg_noise_schedule_sigma_at(const dpg_noise_schedule* s, uint64_t epoch);
DPG_API dpg_status dpg_schedule_noise(dpg_noise_schedule* s, uint64_t epoch, dpg_optimizer* opt, double* sigma);

/* RDP accountant of the subsampled Gaussian mechanism (reference SPEC.md:331-389; spec-only in
 * the reference): integer orders (default 2..64, 128, 256), per-step RDP in log space,
 * additive composition over the recorded (sigma, q, steps), epsilon = min_a rdp(a) + ln(1/delta)/(a-1),
 * and calibration of sigma to a target epsilon by bisection (tolerance 1e-3). */
typedef struct dpg_accountant dpg_accountant;
DPG_API dpg_status dpg_rdp_subsampled_gaussian(double q, double sigma, int alpha, double* out);
DPG_API dpg_status dpg_accountant_create(const int* orders, int n, dpg_accountant** out);
DPG_API void dpg_accountant_destroy(dpg_accountant* a);
DPG_API int dpg_accountant_num_orders(const dpg_accountant* a);
DPG_API dpg_status dpg_accountant_step(dpg_accountant* a, double sigma, double q, int64_t steps);
DPG_API dpg_status dpg_accountant_rdp(const dpg_accountant* a, int* orders, double* curve);
DPG_API dpg_status dpg_accountant_epsilon(const dpg_accountant* a, double delta, double* eps, int* best_order);
DPG_API dpg_status dpg_get_noise_multiplier(double target_eps, double delta, double q, int64_t steps,
                                            double sigma_min, double sigma_max, double* sigma);

/* GradSampleRecord export (Appendix D inspection): parameter `param`'s
 * [b, ...param] per-sample gradients of the pending batch, copied to host (synchronous). */
DPG_API dpg_status dpg_grad_sample_export(const dpg_optimizer* opt, int param, float* host, int64_t capacity);

/* ======================================================================================
 * Diagnostics (no reference counterpart): unit test of the TMA-fed tcgen05 GEMM core that the
 * convolution contractions are built on. D[m][n] = sum_k A[m][k] B[n][k], row-major fp32 device
 * buffers, 3xTF32; bn in {32, 64, 128} output columns per tile, bk in {16, 32} K per stage
 * (K a multiple of 4). bk = -32: b holds B transposed ([k][n] row-major) and lands as an
 * MN-major B tile (bn in {32, 64, 96, 192}). */
DPG_API dpg_status dpg_tg_gemm_selftest(dpg_ctx* ctx, const float* a, const float* b, float* d,
                                        int64_t m, int64_t n, int64_t k, int bn, int bk);
/* The same with the K blocks split over a thread-block cluster of ck CTAs (1, 2, 4) whose
 * partials are summed through distributed shared memory (bk 32, K-major B, bn 32 or 64). */
DPG_API dpg_status dpg_tg_gemm_selftest_split(dpg_ctx* ctx, const float* a, const float* b, float* d,
                                              int64_t m, int64_t n, int64_t k, int bn, int ck);

#ifdef __cplusplus
}
#endif

#endif /* DPG_H */
