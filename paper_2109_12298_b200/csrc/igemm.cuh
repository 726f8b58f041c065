// igemm.cuh — tiled SIMT implicit GEMM used by the first (CUDA-core) path of every contraction
// on the step: conv forward / dgrad, per-sample conv and linear gradients, split-K clipped sums.
//
//   C[z][m][n] = sum_k A(z, m, k) * B(z, k, n)
//
// A problem type `Prob` supplies the operand gathers (implicit im2col lives there), the sizes
// and the epilogue. The K loop runs in ascending k inside every thread, so with
// Prob::kExact the per-output accumulation is the reference's sequential `acc += a * b`
// (two roundings, tensor.hpp:324-336) and reproduces its bits; otherwise FFMA is used.
//
// Tiles are staged through shared memory with a register prefetch of the next k-tile;
// 256 threads, each owning a (BM/16) x (BN/16) sub-tile strided by 16 so that stores along n
// coalesce.
#pragma once

#include "dpg_device.cuh"

namespace dpg {

template <int BM, int BN, int BK, class Prob>
__global__ void __launch_bounds__(256) igemm_kernel(const Prob p) {
  pdl_wait();
  constexpr int TM = BM / 16, TN = BN / 16;
  constexpr int A_PER = (BM * BK + 255) / 256, B_PER = (BK * BN + 255) / 256;
  __shared__ float As[BK][BM + 1];
  __shared__ float Bs[BK][BN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int z = blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t M = p.M, N = p.N, K = p.K;

  float ra[A_PER], rb[B_PER];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int t = 0; t < A_PER; ++t) {
      const int i = tid + t * 256;
      int mm, kk;
      if (Prob::kAMajorM) { mm = i % BM; kk = i / BM; } else { mm = i / BK; kk = i % BK; }
      float v = 0.f;
      if (i < BM * BK && m0 + mm < M && k0 + kk < K) v = p.a(z, m0 + mm, k0 + kk);
      ra[t] = v;
    }
#pragma unroll
    for (int t = 0; t < B_PER; ++t) {
      const int i = tid + t * 256;
      int kk, nn;
      if (Prob::kBMajorN) { nn = i % BN; kk = i / BN; } else { nn = i / BK; kk = i % BK; }
      float v = 0.f;
      if (i < BK * BN && k0 + kk < K && n0 + nn < N) v = p.b(z, k0 + kk, n0 + nn);
      rb[t] = v;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int t = 0; t < A_PER; ++t) {
      const int i = tid + t * 256;
      if (i < BM * BK) {
        int mm, kk;
        if (Prob::kAMajorM) { mm = i % BM; kk = i / BM; } else { mm = i / BK; kk = i % BK; }
        As[kk][mm] = ra[t];
      }
    }
#pragma unroll
    for (int t = 0; t < B_PER; ++t) {
      const int i = tid + t * 256;
      if (i < BK * BN) {
        int kk, nn;
        if (Prob::kBMajorN) { nn = i % BN; kk = i / BN; } else { nn = i / BK; kk = i % BK; }
        Bs[kk][nn] = rb[t];
      }
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = p.init(z, m0 + ty + 16 * i, n0 + tx + 16 * j);

  load(0);
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    stash();
    __syncthreads();
    if (k0 + BK < K) load(k0 + BK);  // prefetch next tile while this one is consumed
    const int kmax = (K - k0) < BK ? int(K - k0) : BK;
    if (kmax == BK) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            if (Prob::kExact) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
            else acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
          }
      }
    } else {
      for (int kk = 0; kk < kmax; ++kk) {
        float a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            if (Prob::kExact) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
            else acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
          }
      }
    }
    __syncthreads();
  }
  p.template epilogue<TM, TN>(z, m0, n0, tx, ty, acc);
}

template <int BM, int BN, int BK, class Prob>
void launch_igemm(dpg_ctx* ctx, const Prob& p, int64_t batches) {
  dim3 grid((unsigned)((p.N + BN - 1) / BN), (unsigned)((p.M + BM - 1) / BM), (unsigned)batches);
  ::dpg::launch_pdl(igemm_kernel<BM, BN, BK, Prob>, grid, 256, 0, ctx->stream, p);
  DPG_LAUNCH_CHECK(ctx);
}

// Epilogue helper: per-thread sum of squares (double) of the stored values, reduced per CTA
// into sq_part[tile * b + z] — one norm-partial row per output tile (deterministic).
template <int TM, int TN>
__device__ __forceinline__ void tile_sq_store(double local, double* sq_part, int64_t b, int z) {
  __shared__ double red[8];
  const double t = block_sum<256>(local, red);
  if (threadIdx.x == 0 && sq_part) {
    const int64_t tile = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    sq_part[tile * b + z] = t;
  }
}

}  // namespace dpg
