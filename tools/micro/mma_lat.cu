// Microbenchmark: latency of a chain of tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) issued by one
// thread with smem operands, committed to an mbarrier and waited on; repeated.
#include <cstdio>
#include <cstdint>
#include "tc_gemm.cuh"
using namespace dpg::tc;

template <int BN>
__global__ void __launch_bounds__(128) mma_lat(int nmma, int reps, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;                  // 128 x 128 B
  uint8_t* b = smem + 128 * 128;      // BN x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(b + BN * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + BN) * 32; i += 128) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 97);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(tmem_cols<BN>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (tid == 0) {
      tc_fence_after();
      for (int i = 0; i < nmma; ++i)
        mma_tf32(tmem, sw128_desc(smem_u32(a) + (i & 3) * 32), sw128_desc(smem_u32(b) + (i & 3) * 32), idesc_tf32(BN), i > 0 ? 1u : 0u);
      mma_commit(bar);
    }
    mbar_wait(bar, r & 1);
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / reps;
  tc_fence_before(); __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols<BN>()));
}

int main() {
  long long* d; cudaMalloc(&d, sizeof(long long) * 1024);
  long long h[1024];
  for (int bn : {32, 64, 128}) {
    for (int nmma : {1, 3, 12, 48}) {
      for (int grid : {1, 148}) {
        const int smem = 1024 + (128 + bn) * 128 + 64;
        if (bn == 32) { cudaFuncSetAttribute(mma_lat<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); mma_lat<32><<<grid, 128, smem>>>(nmma, 200, d); }
        if (bn == 64) { cudaFuncSetAttribute(mma_lat<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); mma_lat<64><<<grid, 128, smem>>>(nmma, 200, d); }
        if (bn == 128) { cudaFuncSetAttribute(mma_lat<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); mma_lat<128><<<grid, 128, smem>>>(nmma, 200, d); }
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
        printf("BN=%3d nmma=%2d grid=%3d: %lld cycles per chain (%.1f per MMA) %s\n", bn, nmma, grid, h[0], (double)h[0] / nmma, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
