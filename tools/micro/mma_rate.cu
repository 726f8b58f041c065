// tcgen05.mma.kind::tf32 issue rate by shape: a chain of 96 MMAs (M = 128, N = BN, K = 8) by one
// thread, A from shared memory (SS) or from TMEM (TS), committed and waited; cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2109_12298_b200/csrc tools/micro/mma_rate.cu -o tools/micro/mma_rate
#include <cstdio>

#include "tg_gemm.cuh"

using namespace dpg::tg;

template <int BN, bool TS>
__global__ void __launch_bounds__(128) rate(int nmma, int reps, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const uint32_t a = su32(smem), b = a + 128 * 128;
  const uint32_t bar = b + BN * 128;
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 128 * 128 + BN * 128 + 8);
  for (int i = threadIdx.x; i < (128 + BN) * 32; i += 128) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int r = 0; r < reps; ++r) {
      for (int i = 0; i < nmma; ++i) {
        if (TS)
          mma_tf32_ts(tmem, tmem + 256 + (i & 3) * 8, KLay<32>::desc(b + (i & 3) * 32), idesc_tf32(BN), i > 0);
        else
          mma_tf32(tmem, KLay<32>::desc(a + (i & 3) * 32), KLay<32>::desc(b + (i & 3) * 32), idesc_tf32(BN), i > 0);
      }
      mma_commit(bar);
      mbar_wait(bar, r & 1);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int BN, bool TS>
void run(long long* d) {
  const int smem = 1024 + (128 + BN) * 128 + 64;
  cudaFuncSetAttribute(rate<BN, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 148}) {
    rate<BN, TS><<<grid, 128, smem>>>(96, 50, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, sizeof(long long), cudaMemcpyDeviceToHost);
    const double per = (double)h / 96;
    printf("%s N=%3d grid=%3d: %.1f cycles per MMA, %.0f MAC/clk/SM %s\n", TS ? "TS" : "SS", BN, grid, per,
           128.0 * BN * 8 / per, cudaGetErrorString(e));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 256);
  run<32, false>(d); run<64, false>(d); run<128, false>(d); run<256, false>(d);
  run<32, true>(d); run<64, true>(d); run<128, true>(d); run<256, true>(d);
  return 0;
}
