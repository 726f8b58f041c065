// Timeline of the TMA-fed GEMM core (tg_gemm.cuh) on one conv-like shape: CTA 0's per-stage
// globaltimer stamps (producer issue, stage landed, converted, MMA start, tile handed to the
// epilogue, epilogue done), to see which role bounds a stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DDPG_TG_TRACE -I include \
//        -I paper_2109_12298_b200/csrc tools/micro/tg_trace.cu -o tools/micro/tg_trace
#include <cstdio>
#include <vector>

#include "tg_gemm.cuh"

using namespace dpg::tg;

template <int BN, int BK>
struct G {
  static constexpr bool kScaleA = false, kScaleB = false, kCtaReduce = false;
  float* d;
  int M, N, K;
  __device__ int nkb(int) const { return (K + BK - 1) / BK; }
  __device__ uint32_t stage_bytes() const { return (uint32_t)((BM + BN) * BK * 4); }
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t bar, int mt, int nt, int, const CUtensorMap* ma,
                        const CUtensorMap* mb) const {
    tma2(sa, ma, bar, kb * BK, mt * BM);
    tma2(sb, mb, bar, kb * BK, nt * BN);
  }
  __device__ float scale(int, int, int, int) const { return 1.f; }
  __device__ void epilogue(int mt, int nt, int, int row, int c0, const float (&v)[16], double&) const {
    const int m = mt * BM + row;
    if (m >= M) return;
    float* o = d + (int64_t)m * N + nt * BN + c0;
#pragma unroll
    for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  }
  __device__ void finish(int, int, int, double) const {}
};

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int M = 32768, N = 64, K = argc > 1 ? atoi(argv[1]) : 288;
  constexpr int BN = 64, BK = 32, ST = stages_for<BN, BK>();
  float *a, *b, *d;
  cudaMalloc(&a, sizeof(float) * M * K);
  cudaMalloc(&b, sizeof(float) * N * K);
  cudaMalloc(&d, sizeof(float) * M * N);
  cudaMemset(a, 0, sizeof(float) * M * K);
  cudaMemset(b, 0, sizeof(float) * N * K);
  Enc enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap ma, mb;
  cuuint64_t da[2] = {(cuuint64_t)K, (cuuint64_t)M}, db[2] = {(cuuint64_t)K, (cuuint64_t)N}, st[1] = {(cuuint64_t)K * 4};
  cuuint32_t ba[2] = {BK, BM}, bb[2] = {BK, BN}, es[2] = {1, 1};
  enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, da, st, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE, KLay<BK>::TMA_SWIZZLE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b, db, st, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, KLay<BK>::TMA_SWIZZLE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  G<BN, BK> p{d, M, N, K};
  Tiles tiles{M / BM, 1, 1};
  const int smem = Smem<BN, BK, ST>::TOTAL;
  cudaFuncSetAttribute(tg_kernel<BN, BK, ST, G<BN, BK>>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int on = 1;
  cudaMemcpyToSymbol(g_tg_trace_on, &on, sizeof(int));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    tg_kernel<BN, BK, ST, G<BN, BK>><<<148, kThreads2, smem>>>(ma, mb, p, tiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %.1f us (%s) ST=%d\n", rep, ms * 1e3, cudaGetErrorString(cudaGetLastError()), ST);
  }
  std::vector<unsigned long long> tr(8 * 256);
  cudaMemcpyFromSymbol(tr.data(), g_tg_trace, sizeof(unsigned long long) * 8 * 256);
  const unsigned long long t0 = tr[0];
  const int nkb = (K + BK - 1) / BK;
  const int its = nkb * ((M / BM + 147) / 148);
  printf("it: issue landed converted mma_start (ns from first issue)\n");
  for (int i = 0; i < its && i < 64; ++i)
    printf("%3d: %7lld %7lld %7lld %7lld\n", i, (long long)(tr[0 * 256 + i] - t0), (long long)(tr[1 * 256 + i] - t0),
           (long long)(tr[2 * 256 + i] - t0), (long long)(tr[3 * 256 + i] - t0));
  for (int j = 0; j < 3; ++j)
    printf("tile %d: tfull %lld epi_done %lld\n", j, (long long)(tr[4 * 256 + j] - t0), (long long)(tr[5 * 256 + j] - t0));
  return 0;
}
