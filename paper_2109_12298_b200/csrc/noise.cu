// noise.cu — Gaussian noise + averaged SGD update, fused (north-star subsystem 4).
//
// Reference: add_noise (optimizer.hpp:120-133) -> gaussian (tensor.hpp:343-354) ->
// RngStream::normal (rng.cpp:40-53, Box-Muller in double), then finish_step
// (optimizer.hpp:256-271): g = noised * (1/E), w = w - g * lr in fp32.
//
// The device stream is counter-based Philox4x32-10 (Salmon et al., Random123) keyed by the
// 64-bit noise seed with counter (element pair, step): every rank and every replay draws the
// same value for the same (seed, step, element) with no state to carry, which is what lets the
// sample-sharded step add noise once after the all-reduce without a broadcast. Box-Muller uses
// the reference's uniform construction: u1 = ((x >> 11) + 1) * 2^-53 in (0, 1],
// u2 = (y >> 11) * 2^-53 in [0, 1); element 2q gets r cos(theta), 2q+1 gets r sin(theta).
#include <algorithm>

#include "step_common.cuh"

namespace dpg {

// Graph replays keep the Philox step on the device: every CTA reads it first, and the last CTA
// to take a ticket (self-resetting counter) writes step + 1 for the next replay — no host-to-device
// copy per step. Called by every thread of the CTA before any early return.
__device__ __forceinline__ void advance_step(uint64_t* step_ptr, uint64_t step, unsigned long long* ticket) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ticket, 1ull) == gridDim.x - 1) {
      atomicExch(ticket, 0ull);
      *step_ptr = step + 1;
    }
  }
}

// Multi-rank steps carry one status lane after the L clipped-sum elements: each rank writes 1 when
// it has an error pending (non-finite per-sample gradient, bad target / index), the exchange
// sums the lanes with the clipped sums, and every rank skips the update when the sum is
// non-zero — the reference's step throws before touching any parameter, on every rank alike.
__global__ void status_lane_kernel(float* __restrict__ lane, const DeviceErr* err) {
  pdl_wait();
  if (threadIdx.x == 0) *lane = error_pending(err) ? 1.f : 0.f;
}

void launch_status_lane(dpg_ctx* ctx, float* lane) {
  ::dpg::launch_pdl(status_lane_kernel, 1u, 32, 0, ctx->stream, lane, (const DeviceErr*)ctx->dev_err);
  DPG_LAUNCH_CHECK(ctx);
}

// true when the step must not update: a local error, or (status lane) an error on another rank,
// which is then recorded locally so the host surfaces it here too
__device__ __forceinline__ bool skip_update(DeviceErr* err, float status) {
  if (error_pending(err)) return true;
  if (status != 0.f) {
    report_error(err, err_key(ERR_STAGE_REMOTE, 0, 0), 0);
    return true;
  }
  return false;
}

// One thread per element pair. If an earlier stage flagged an error (NumericError etc.) the
// update is skipped: the reference throws before touching the parameters.
__global__ void __launch_bounds__(256) noise_update_kernel(
    float* __restrict__ params, const float* __restrict__ summed, float* __restrict__ grad,
    int64_t n, double std_dev, float inv_e, float lr, uint64_t seed, uint64_t step,
    const float* __restrict__ injected, uint64_t* step_ptr, DeviceErr* err,
    unsigned long long* advance, const float* status) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = 2 * q;
  if (step_ptr) step = *step_ptr;
  if (advance) advance_step(step_ptr, step, advance);  // after every CTA has read it
  if (i0 >= n) return;
  if (skip_update(err, status ? *status : 0.f)) return;
  float nz[2] = {0.f, 0.f};
  if (injected) {
    nz[0] = injected[i0];
    if (i0 + 1 < n) nz[1] = injected[i0 + 1];
  } else if (std_dev != 0.0) {
    double z0, z1;
    normal_pair(seed, step, (uint64_t)q, z0, z1);
    nz[0] = (float)(z0 * std_dev);
    nz[1] = (float)(z1 * std_dev);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int64_t i = i0 + k;
    if (i >= n) break;
    const float noised = (injected || std_dev != 0.0) ? __fadd_rn(summed[i], nz[k]) : summed[i];
    const float g = __fmul_rn(noised, inv_e);
    params[i] = __fsub_rn(params[i], __fmul_rn(g, lr));
    if (grad) grad[i] = g;
  }
}

void launch_noise_update(dpg_ctx* ctx, float* params, const float* summed, float* grad, int64_t n,
                         double sigma, double c, double expected_batch, double lr, uint64_t seed,
                         uint64_t step, const float* injected, uint64_t* step_ptr,
                         unsigned long long* advance, const float* status) {
  if (n == 0) return;
  const double std_dev = sigma * c;
  const float denom = (float)expected_batch;
  const float inv_e = 1.0f / denom;  // T(1) / denom (optimizer.hpp:259, 264)
  const int64_t pairs = (n + 1) / 2;
  ::dpg::launch_pdl(noise_update_kernel, (unsigned)((pairs + 255) / 256), 256, 0, ctx->stream, 
      params, summed, grad, n, std_dev, inv_e, (float)lr, seed, step, injected, step_ptr, ctx->dev_err, advance,
      status);
  DPG_LAUNCH_CHECK(ctx);
}

// ------------------------------------------------------------------ exchange over peer memory
// The sample-sharded step's one exchange (an all-reduce of the clipped sum)
// fused into the noise update: every rank maps its peers' optimizer arenas (CUDA IPC; NVLink
// P2P between GPUs), publishes "my clipped sum of epoch e is complete" in a flag, and the
// update kernel sums the W clipped sums straight from peer memory in rank order 0..W-1 — the
// same order on every rank, so the parameters stay bitwise identical without a broadcast.
// Epoch e = Philox step + 1 (identical on every rank, strictly increasing; flags start at 0).
//   xch_signal      flag[SIG] = e (release, system scope) after the clipped-sum kernels
//   noise (p2p)     wait flag[SIG] >= e on every rank; sum; noise; update; the last CTA to finish
//                   reading sets flag[ACK] = e
//   xch_complete    wait flag[ACK] >= e on every rank (nobody still reads my clipped sum), then
//                   copy the reduced sum into `summed` (the NCCL path's in-place result) — after
//                   which the next step may overwrite it
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Bounded: a peer that never arrives (a rank died, or ranks disagree on the number of steps)
// traps after 120 s, failing the launch with an error instead of hanging the device.
__device__ __forceinline__ void wait_all(const PeerSet& ps, int slot, unsigned long long e) {
  const unsigned long long t0 = global_ns();
  for (int r = 0; r < ps.world; ++r)
    while (ld_acquire_sys(ps.flags[r] + slot) < e) {
      __nanosleep(256);
      if (global_ns() - t0 > 120ull * 1000000000ull) __trap();
    }
}

__global__ void xch_signal_kernel(PeerSet ps, uint64_t step, const uint64_t* step_ptr) {
  pdl_wait();
  if (step_ptr) step = *step_ptr;
  __threadfence_system();
  st_release_sys(ps.flags[ps.rank] + PeerSet::kSig, step + 1);
}

__global__ void __launch_bounds__(256) noise_update_p2p_kernel(
    float* __restrict__ params, float* __restrict__ reduced, float* __restrict__ grad, int64_t n,
    double std_dev, float inv_e, float lr, uint64_t seed, uint64_t step, const float* __restrict__ injected,
    const uint64_t* step_ptr, DeviceErr* err, PeerSet ps) {
  pdl_wait();
  if (step_ptr) step = *step_ptr;
  const unsigned long long e = step + 1;
  __shared__ float status;  // sum of the W status lanes (element n of every clipped-sum buffer)
  if (threadIdx.x == 0) {
    wait_all(ps, PeerSet::kSig, e);
    float st = 0.f;
    for (int r = 0; r < ps.world; ++r) st += __ldcg(ps.summed[r] + n);
    status = st;
    if (blockIdx.x == 0) reduced[n] = st;
  }
  __syncthreads();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = 2 * q;
  if (i0 < n) {
    float s[2] = {0.f, 0.f};
    for (int r = 0; r < ps.world; ++r) {
      s[0] += __ldcg(ps.summed[r] + i0);
      if (i0 + 1 < n) s[1] += __ldcg(ps.summed[r] + i0 + 1);
    }
    float nz[2] = {0.f, 0.f};
    if (injected) {
      nz[0] = injected[i0];
      if (i0 + 1 < n) nz[1] = injected[i0 + 1];
    } else if (std_dev != 0.0) {
      double z0, z1;
      normal_pair(seed, step, (uint64_t)q, z0, z1);
      nz[0] = (float)(z0 * std_dev);
      nz[1] = (float)(z1 * std_dev);
    }
    const bool skip = skip_update(err, status);  // still takes part in the exchange: peers wait on us
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int64_t i = i0 + k;
      if (i >= n) break;
      reduced[i] = s[k];
      if (skip) continue;
      const float noised = (injected || std_dev != 0.0) ? __fadd_rn(s[k], nz[k]) : s[k];
      const float g = __fmul_rn(noised, inv_e);
      params[i] = __fsub_rn(params[i], __fmul_rn(g, lr));
      if (grad) grad[i] = g;
    }
  }
  __syncthreads();  // this CTA's peer reads are done
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned long long* cnt = ps.flags[ps.rank] + PeerSet::kCount;
    if (atomicAdd(cnt, 1ull) % gridDim.x == gridDim.x - 1) {
      __threadfence_system();
      st_release_sys(ps.flags[ps.rank] + PeerSet::kAck, e);
    }
  }
}

__global__ void xch_complete_kernel(PeerSet ps, const float* __restrict__ reduced, float* __restrict__ summed,
                                    int64_t n, uint64_t step, uint64_t* step_ptr, unsigned long long* advance) {
  pdl_wait();
  if (step_ptr) step = *step_ptr;
  if (advance) advance_step(step_ptr, step, advance);
  if (threadIdx.x == 0) wait_all(ps, PeerSet::kAck, step + 1);
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    summed[i] = reduced[i];  // (element n: the summed status lane)
}

void launch_noise_update_p2p(dpg_ctx* ctx, const PeerSet& ps, float* params, float* summed, float* reduced,
                             float* grad, int64_t n, double sigma, double c, double expected_batch, double lr,
                             uint64_t seed, uint64_t step, const float* injected, uint64_t* step_ptr,
                             unsigned long long* advance) {
  ::dpg::launch_pdl(xch_signal_kernel, 1u, 32, 0, ctx->stream, ps, step, step_ptr);
  DPG_LAUNCH_CHECK(ctx);
  const double std_dev = sigma * c;
  const float inv_e = 1.0f / (float)expected_batch;
  const int64_t pairs = std::max<int64_t>(1, (n + 1) / 2);
  ::dpg::launch_pdl(noise_update_p2p_kernel, (unsigned)((pairs + 255) / 256), 256, 0, ctx->stream, params,
                    reduced, grad, n, std_dev, inv_e, (float)lr, seed, step, injected, step_ptr, ctx->dev_err, ps);
  DPG_LAUNCH_CHECK(ctx);
  ::dpg::launch_pdl(xch_complete_kernel, (unsigned)std::min<int64_t>(kNumSMs, (n + 255) / 256 + 1), 256, 0,
                    ctx->stream, ps, (const float*)reduced, summed, n, step, step_ptr, advance);
  DPG_LAUNCH_CHECK(ctx);
}

__global__ void gaussian_kernel(float* __restrict__ out, int64_t n, double std_dev, uint64_t seed,
                                uint64_t step) {
  pdl_wait();
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = 2 * q;
  if (i0 >= n) return;
  double z0, z1;
  normal_pair(seed, step, (uint64_t)q, z0, z1);
  out[i0] = (float)(z0 * std_dev);
  if (i0 + 1 < n) out[i0 + 1] = (float)(z1 * std_dev);
}

void launch_gaussian(dpg_ctx* ctx, float* out, int64_t n, double std_dev, uint64_t seed,
                     uint64_t step) {
  if (n == 0) return;
  if (std_dev == 0.0) {
    DPG_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)n, ctx->stream));
    return;
  }
  const int64_t pairs = (n + 1) / 2;
  ::dpg::launch_pdl(gaussian_kernel, (unsigned)((pairs + 255) / 256), 256, 0, ctx->stream, out, n, std_dev, seed, step);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace dpg
