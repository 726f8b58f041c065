// Microbenchmark: cost per stage of the producer -> MMA-thread pipeline skeleton (no loads, no
// MMAs): producers store a stage, fence.proxy.async, arrive on full[s]; the MMA thread waits
// full[s] and releases the slot (tcgen05.commit or a plain arrive); producers wait empty[s].
// Flags: 1 = skip fence, 2 = per-warp arrive (count 8), 4 = plain arrive instead of commit,
//        8 = skip the stores, 16 = one __syncthreads-style CTA barrier instead of mbarriers
#include <cstdio>
#include <cstdint>
#include "tc_gemm.cuh"
using namespace dpg::tc;

__global__ void __launch_bounds__(416, 1) skel(int nst, int flags, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int NS = 6, STAGE = 24576;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * STAGE);
  uint64_t* empty = full + NS;
  uint32_t* slot = reinterpret_cast<uint32_t*>(empty + NS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 12) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], (flags & 2) ? 8 : 256);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t tmem = *slot;
  long long t0 = clock64();
  if (flags & 16) {
    for (int g = 0; g < nst; ++g) {
      if (warp < 8 && !(flags & 8)) {
        uint8_t* st = smem + (g % 2) * STAGE;
        for (int i = 0; i < 6; ++i) *reinterpret_cast<uint4*>(st + ((tid + 256 * i) * 16) % STAGE) = make_uint4(g, i, tid, 0);
      }
      if (!(flags & 1)) fence_proxy_async();
      __syncthreads();
      if (tid == 0) mma_commit(&empty[g % 2]);
    }
  } else if (warp < 8) {
    for (int g = 0; g < nst; ++g) {
      const int s = g % NS;
      if (g >= NS) mbar_wait(&empty[s], ((g / NS) - 1) & 1);
      if (!(flags & 8)) {
        uint8_t* st = smem + s * STAGE;
        for (int i = 0; i < 6; ++i) *reinterpret_cast<uint4*>(st + ((tid + 256 * i) * 16) % STAGE) = make_uint4(g, i, tid, 0);
      }
      if (!(flags & 1)) fence_proxy_async();
      if (flags & 2) {
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      }
    }
  } else if (warp == 12 && lane == 0) {
    for (int g = 0; g < nst; ++g) {
      const int s = g % NS;
      mbar_wait(&full[s], (g / NS) & 1);
      tc_fence_after();
      if (flags & 4) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      else mma_commit(&empty[s]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / nst;
  if (warp == 12) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  long long h[148];
  const int smem = 6 * 24576 + 2048;
  cudaFuncSetAttribute(skel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int flags : {0, 1, 2, 3, 4, 5, 6, 7, 8, 15, 16, 17, 24}) {
    skel<<<148, 416, smem>>>(2000, flags, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("flags=%2d: %lld cycles/stage (max over CTAs) %s\n", flags, mx, cudaGetErrorString(e));
  }
  return 0;
}
