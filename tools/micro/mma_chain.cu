// Does splitting one accumulate chain over several independent TMEM accumulators overlap MMAs?
#include <cstdio>
#include <cstdint>
#include "tc_gemm.cuh"
using namespace dpg::tc;

template <int BN>
__global__ void __launch_bounds__(128) chain(int nmma, int nacc, int reps, long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem; uint8_t* b = smem + 128 * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(b + BN * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + BN) * 32; i += 128) reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 97);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  uint64_t ad[4], bd[4];
  for (int k = 0; k < 4; ++k) { ad[k] = sw128_desc(smem_u32(a) + 32 * k); bd[k] = sw128_desc(smem_u32(b) + 32 * k); }
  const uint32_t id = idesc_tf32(BN);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (tid == 0) {
      tc_fence_after();
#pragma unroll 4
      for (int i = 0; i < nmma; ++i) {
        const int acc = i % nacc;
        mma_tf32(tmem + acc * BN, ad[i & 3], bd[i & 3], id, i >= nacc ? 1u : 0u);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, r & 1);
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  tc_fence_before(); __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  long long* c; cudaMalloc(&c, 8 * 256); long long h;
  for (int bn : {64, 128}) for (int nacc : {1, 2, 3, 4}) for (int nmma : {12, 48}) {
    const int smem = 1024 + (128 + bn) * 128 + 64;
    if (bn == 64) { cudaFuncSetAttribute(chain<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); chain<64><<<1, 128, smem>>>(nmma, nacc, 100, c); }
    else { cudaFuncSetAttribute(chain<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); chain<128><<<1, 128, smem>>>(nmma, nacc, 100, c); }
    cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("BN=%3d nacc=%d nmma=%2d: %lld cycles (%.1f / MMA) %s\n", bn, nacc, nmma, h, (double)h / nmma, cudaGetErrorString(e));
  }
  // two CTAs per SM sharing the tensor core
  return 0;
}
