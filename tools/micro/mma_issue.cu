// Per-MMA cost vs N with a fully unrolled issue loop (descriptors derived from two base
// registers), alone on the SM and with 2 CTAs per SM sharing the tensor core.
#include <cstdio>
#include <cstdint>
#include "tc_gemm.cuh"
using namespace dpg::tc;

template <int BN, int NMMA, int MODE>
__global__ void __launch_bounds__(128) issue_test(int reps, long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem; uint8_t* b = smem + 128 * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(b + BN * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + BN) * 32; i += 128) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 97);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(tmem_cols<BN>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = *slot;
  if (MODE == 1) tmem = __shfl_sync(0xffffffffu, tmem, 0);
  if (MODE == 2) tmem = 0;
  const uint64_t a0 = sw128_desc(smem_u32(a)), b0 = sw128_desc(smem_u32(b));
  constexpr uint32_t id = idesc_tf32(BN);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (tid < 32) {
      if (tid == 0) {
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < NMMA; ++i) mma_tf32(tmem, a0 + 2 * (i & 3), b0 + 2 * (i & 3), id, i > 0 ? 1u : 0u);
        mma_commit(bar);
      }
      __syncwarp();
    }
    mbar_wait(bar, r & 1);
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  tc_fence_before(); __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols<BN>()));
}

template <int BN, int NMMA, int MODE = 0>
void run(int grid, long long* c) {
  const int smem = 1024 + (128 + BN) * 128 + 64;
  cudaFuncSetAttribute(issue_test<BN, NMMA, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  issue_test<BN, NMMA, MODE><<<grid, 128, smem>>>(200, c);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296]; cudaMemcpy(h, c, 8 * grid, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mode=%d BN=%3d nmma=%2d grid=%3d: %lld cycles max (%.1f / MMA, %.0f MAC/clk/CTA) %s\n", MODE, BN, NMMA, grid, mx, (double)mx / NMMA,
         128.0 * BN * 8 * NMMA / mx, cudaGetErrorString(e));
}

int main() {
  long long* c; cudaMalloc(&c, 8 * 296);
  run<32, 12>(1, c); run<32, 48>(1, c);
  run<64, 12>(1, c); run<64, 48>(1, c);
  run<128, 12>(1, c); run<128, 48>(1, c);
  run<256, 12>(1, c); run<256, 48>(1, c);
  run<64, 48>(296, c); run<128, 48>(296, c); run<256, 48>(296, c);
  run<32, 48, 1>(1, c); run<64, 48, 1>(1, c); run<128, 48, 1>(1, c); run<256, 48, 1>(1, c);
  run<32, 48, 2>(1, c); run<64, 48, 2>(1, c); run<128, 48, 2>(1, c); run<256, 48, 2>(1, c);
  run<64, 48, 1>(296, c); run<128, 48, 1>(296, c);
  return 0;
}
