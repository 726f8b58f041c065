// tcgen05.mma.kind::tf32 TS (A in TMEM) issue rate under interference: one thread issues chains of
// 12 MMAs (M = 128, N = BN, K = 8) walking a 6-stage ring of B in shared memory and of A in TMEM
// (as tg_gemm.cuh does); optionally 4 warps keep writing TMEM (tcgen05.st, converter-like) and/or
// shared memory (converter-like LDS/STS) meanwhile. Cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2109_12298_b200/csrc tools/micro/mma_rate2.cu -o tools/micro/mma_rate2
#include <cstdio>

#include "tg_gemm.cuh"

using namespace dpg::tg;

template <int BN>
__global__ void __launch_bounds__(160) rate(int mode, int reps, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  constexpr int BB = BN * 128;  // B stage bytes (32 fp32 per row)
  const uint32_t b = su32(smem);
  const uint32_t bar = b + 6 * 2 * BB;
  volatile int* stop = reinterpret_cast<volatile int*>(smem + 6 * 2 * BB + 16);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 6 * 2 * BB + 32);
  for (int i = threadIdx.x; i < 6 * 2 * BB / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    *stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        const int s = r % 6;
        const uint32_t ahi = tmem + 2 * BN + s * 64, alo = ahi + 32;
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t bd = b + s * 2 * BB + kk * 32;
          mma_tf32_ts(tmem, alo + kk * 8, KLay<32>::desc(bd), idesc_tf32(BN), (r | kk) > 0);
          mma_tf32_ts(tmem, ahi + kk * 8, KLay<32>::desc(bd + BB), idesc_tf32(BN), 1u);
          mma_tf32_ts(tmem, ahi + kk * 8, KLay<32>::desc(bd), idesc_tf32(BN), 1u);
        }
        mma_commit(bar);
        mbar_wait(bar, r & 1);
      }
      out[blockIdx.x] = (clock64() - t0) / reps;
      *stop = 1;
    }
  } else {
    // interference warps 1-4: TMEM lanes 32 (w % 4) ...
    const int q = warp & 3;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * q) << 16);
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = 0;
    int s = 0;
    while (!*stop) {
      if (mode & 1) {  // tcgen05.st 64 columns into a stage's A slot
        for (int h = 0; h < 4; ++h) tmem_st16(lane_addr + 2 * BN + ((s + 3) % 6) * 64 + 16 * h, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (mode & 2) {  // LDS + 2 STS of 16 B per thread over a 16 KB region
        uint8_t* base = smem + ((s + 3) % 6) * 2 * BB;
        for (int i = (threadIdx.x - 32) * 16; i < BB; i += 128 * 16) {
          uint4 x;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(su32(base + i)));
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(su32(base + i)), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w));
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(su32(base + BB + i)), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w));
        }
      }
      if (!(mode & 3)) __nanosleep(100);
      s = (s + 1) % 6;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int BN>
void run(long long* d) {
  const int smem = 1024 + 6 * 2 * BN * 128 + 64;
  cudaFuncSetAttribute(rate<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode : {0, 1, 2, 3}) {
    rate<BN><<<148, 160, smem>>>(mode, 200, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("N=%3d mode %d (%s%s): %.1f cycles per MMA %s\n", BN, mode, mode & 1 ? "tmem-st " : "", mode & 2 ? "smem" : "",
           (double)h / 12, cudaGetErrorString(e));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 256);
  run<32>(d);
  run<64>(d);
  run<128>(d);
  return 0;
}
