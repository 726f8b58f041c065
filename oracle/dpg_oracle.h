/*
 * dpg_oracle.h — CPU restatement of the reference DP-SGD step (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for the B200 path. It restates, loop for loop and in the same
 * floating-point association order, the reference C++ implementation under
 * /root/reference/proj/core (dpgrad). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product (libdpg.so) never does.
 *
 * Pinning: tests/test_oracle_vs_reference.py checks every entry point here bit-for-bit
 * against the real reference compiled from its own sources (oracle/ref_shim.cpp ->
 * oracle/_ref/libdpgref.so) and against the SPEC known-answer tests; the committed
 * fixtures in tests/golden/ were generated from the reference by oracle/make_golden.py.
 *
 * Every function is provided for float (suffix _f32) and double (suffix _f64); build with
 * -O2 -ffp-contract=off so that `acc += a * b` stays two roundings, as in the reference's
 * parity build (g++ -O2 -std=c++20, no -march, SURVEY.md §8c "compile-flag hazard").
 */
#ifndef DPG_ORACLE_H
#define DPG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: identical numbering to include/dpg.h (errors.hpp:12-72 classes). */
enum {
  DPGO_OK = 0,
  DPGO_ERR_DIMENSION = 1,
  DPGO_ERR_PARAMETER = 2,
  DPGO_ERR_LIFECYCLE = 3,
  DPGO_ERR_REGISTRY = 4,
  DPGO_ERR_NUMERIC = 5,
};

/* Layer kinds: same order as dpgrad::LayerKind (layers.hpp:19-30). */
enum {
  DPGO_LINEAR = 0,
  DPGO_EMBEDDING = 1,
  DPGO_CONV2D = 2,
  DPGO_LAYER_NORM = 3,
  DPGO_GROUP_NORM = 4,
  DPGO_RELU = 5,
  DPGO_FLATTEN = 6,
};

/* Same field layout as dpg_layer_desc in include/dpg.h (LayerDescriptor, layers.hpp:69-194). */
typedef struct dpgo_layer {
  int32_t kind;
  int32_t has_bias;
  int64_t in_features, out_features;  /* linear */
  int64_t vocab_size, embedding_dim;  /* embedding */
  int64_t in_channels, out_channels, kernel_h, kernel_w, stride, padding; /* conv2d */
  int64_t norm_size, groups; double eps; /* layer_norm / group_norm (not in the restatement) */
} dpgo_layer;

/* ---- RngStream::standard (rng.cpp:15-66): std::mt19937_64 + Box-Muller with a spare ---- */
typedef struct dpgo_rng {
  uint64_t mt[312];
  int mti;
  int has_spare;
  double spare;
} dpgo_rng;

void dpgo_rng_seed(dpgo_rng* r, uint64_t seed);
uint64_t dpgo_rng_next_u64(dpgo_rng* r);
double dpgo_rng_uniform(dpgo_rng* r);
double dpgo_rng_normal(dpgo_rng* r);
uint64_t dpgo_rng_below(dpgo_rng* r, uint64_t n);

/* Error message of the last failing call on this thread. */
const char* dpgo_last_error(void);

#define DPGO_DECLARE(REAL, SFX)                                                                  \
  void dpgo_gaussian##SFX(dpgo_rng* r, int64_t n, double std_dev, REAL* out);                    \
  void dpgo_uniform##SFX(dpgo_rng* r, int64_t n, double lo, double hi, REAL* out);               \
  int64_t dpgo_param_count##SFX(const dpgo_layer* layers, int nlayers);                          \
  int dpgo_build_params##SFX(const dpgo_layer* layers, int nlayers, dpgo_rng* r, REAL* params);  \
  int dpgo_batched_outer##SFX(const REAL* bgr, const REAL* acts, int64_t n, int64_t mid,         \
                              int64_t di, int64_t dj, REAL* out);                                \
  int dpgo_sum_middle##SFX(const REAL* t, int64_t n, int64_t mid, int64_t d, REAL* out);         \
  int dpgo_im2col##SFX(const REAL* x, int64_t b, int64_t ic, int64_t h, int64_t w, int64_t kh,   \
                       int64_t kw, int64_t stride, int64_t pad, REAL* cols);                     \
  int dpgo_rule_linear##SFX(const REAL* acts, const REAL* hw, int64_t b, int64_t mid, int64_t d, \
                            int64_t r, REAL* gw, REAL* gb);                                      \
  int dpgo_rule_conv2d##SFX(const REAL* x, const REAL* hw, int64_t b, int64_t ic, int64_t h,     \
                            int64_t w, int64_t oc, int64_t kh, int64_t kw, int64_t stride,       \
                            int64_t pad, REAL* gw, REAL* gb);                                    \
  int dpgo_rule_embedding##SFX(const REAL* idx, const REAL* hw, int64_t b, int64_t t,            \
                               int64_t vocab, int64_t dim, REAL* out);                           \
  int dpgo_clip_and_sum##SFX(const REAL* const* g, const int64_t* numel, int nparams, int64_t b, \
                             double c, REAL* const* summed, double* norms, double* scales,       \
                             int64_t* num_clipped, int64_t* bad_param, int64_t* bad_sample);     \
  int dpgo_add_noise##SFX(const REAL* summed, int64_t n, double sigma, double c, dpgo_rng* r,     \
                          REAL* out);                                                            \
  int dpgo_dpsgd_step##SFX(const dpgo_layer* layers, int nlayers, const int64_t* in_shape,       \
                           int in_rank, int64_t b, const int64_t* shard_sizes, int nshards,      \
                           REAL* params, const REAL* x, const REAL* targets, double sigma,       \
                           double c, double lr, double expected_batch, uint64_t noise_seed,      \
                           const REAL* injected_noise, REAL* record, REAL* summed, REAL* grad,   \
                           double* norms, double* scales, int64_t* num_clipped, REAL* loss,      \
                           REAL* logits);

DPGO_DECLARE(float, _f32)
DPGO_DECLARE(double, _f64)

#ifdef __cplusplus
}
#endif

#endif /* DPG_ORACLE_H */
