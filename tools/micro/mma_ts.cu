// TS-mode (A in TMEM) vs SS-mode tcgen05.mma.kind::tf32: correctness (same D) and chain latency.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "tc_gemm.cuh"
using namespace dpg::tc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}

template <int BN>
__global__ void __launch_bounds__(128) ts_test(int nmma, int reps, int use_ts, float* dout, long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = smem;              // SW128 128 x 32 fp32
  uint8_t* b = smem + 128 * 128;  // SW128 BN x 32
  uint64_t* bar = reinterpret_cast<uint64_t*>(b + BN * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A[r][k] = tf32((r*7 + k*3) % 13 - 6) * 0.25 ; B[n][k] = ((n*5 + k) % 11 - 5) * 0.5
  for (int r = tid; r < 128; r += 128)
    for (int q = 0; q < 8; ++q) {
      uint4 v;
      uint32_t* pv = &v.x;
      for (int e = 0; e < 4; ++e) { int k = 4 * q + e; pv[e] = to_tf32(((r * 7 + k * 3) % 13 - 6) * 0.25f); }
      *reinterpret_cast<uint4*>(a + sw128_off(r, q)) = v;
    }
  for (int n = tid; n < BN; n += 128)
    for (int q = 0; q < 8; ++q) {
      uint4 v;
      uint32_t* pv = &v.x;
      for (int e = 0; e < 4; ++e) { int k = 4 * q + e; pv[e] = to_tf32(((n * 5 + k) % 11 - 5) * 0.5f); }
      *reinterpret_cast<uint4*>(b + sw128_off(n, q)) = v;
    }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t tA = tmem + 128;  // A operand columns [128, 160)
  // write A into TMEM: row r = 32 warp + lane, columns k
  {
    const int r = 32 * warp + lane;
    for (int k0 = 0; k0 < 32; k0 += 8) {
      uint32_t v[8];
      for (int e = 0; e < 8; ++e) { int k = k0 + e; v[e] = to_tf32(((r * 7 + k * 3) % 13 - 6) * 0.25f); }
      tmem_st8(tA + ((uint32_t)(32 * warp) << 16) + k0, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (tid == 0) {
      tc_fence_after();
      for (int i = 0; i < nmma; ++i) {
        const int kk = i & 3;
        if (use_ts) mma_ts(tmem, tA + 8 * kk, sw128_desc(smem_u32(b) + kk * 32), idesc_tf32(BN), i > 0 ? 1u : 0u);
        else mma_tf32(tmem, sw128_desc(smem_u32(a) + kk * 32), sw128_desc(smem_u32(b) + kk * 32), idesc_tf32(BN), i > 0 ? 1u : 0u);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, rep & 1);
  }
  long long t1 = clock64();
  tc_fence_after();
  if (tid == 0) cyc[0] = (t1 - t0) / reps;
  // read D
  for (int c0 = 0; c0 < BN; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
    for (int j = 0; j < 16; ++j) dout[(32 * warp + lane) * BN + c0 + j] = v[j];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  const int BN = 64;
  float *d1, *d2; long long* c;
  cudaMalloc(&d1, 128 * BN * 4); cudaMalloc(&d2, 128 * BN * 4); cudaMalloc(&c, 64);
  const int smem = 1024 + (128 + BN) * 128 + 64;
  cudaFuncSetAttribute(ts_test<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int nmma : {4, 12, 48}) {
    long long h1, h2;
    ts_test<BN><<<1, 128, smem>>>(nmma, 100, 0, d1, c); cudaDeviceSynchronize(); cudaMemcpy(&h1, c, 8, cudaMemcpyDeviceToHost);
    ts_test<BN><<<1, 128, smem>>>(nmma, 100, 1, d2, c); cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(&h2, c, 8, cudaMemcpyDeviceToHost);
    float a[128 * BN], b[128 * BN];
    cudaMemcpy(a, d1, sizeof a, cudaMemcpyDeviceToHost); cudaMemcpy(b, d2, sizeof b, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (int i = 0; i < 128 * BN; ++i) { md = fmax(md, fabs(a[i] - b[i])); mx = fmax(mx, fabs(a[i])); }
    // reference for one row via host math (nmma slices of k = (i&3)*8..+8)
    double ref00 = 0;
    for (int i = 0; i < nmma; ++i) for (int k = (i & 3) * 8; k < (i & 3) * 8 + 8; ++k) ref00 += (((0 * 7 + k * 3) % 13 - 6) * 0.25) * (((0 * 5 + k) % 11 - 5) * 0.5);
    printf("nmma=%2d SS %lld cyc (%.1f/mma)  TS %lld cyc (%.1f/mma)  max|SS-TS|=%g max|D|=%g D00 ss=%g ts=%g ref=%g %s\n", nmma, h1, (double)h1 / nmma, h2,
           (double)h2 / nmma, md, mx, a[0], b[0], ref00, cudaGetErrorString(e));
  }
  return 0;
}
