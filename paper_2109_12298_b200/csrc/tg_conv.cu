// tg_conv.cu — the TMA-fed tcgen05 contractions (tg_gemm.cuh): tensor-map construction and the
// plain row-major GEMM the core is unit-tested through (dpg_tg_gemm_selftest).
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "tg_gemm.cuh"

namespace dpg {
namespace tg {

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  if (!fn) raise(DPG_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable (driver too old for TMA)");
  return fn;
}
}  // namespace

int max_active_clusters(const void* fn, int smem, int ck, int threads) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int>, int> memo;
  int dev = 0;
  DPG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = memo.find({dev, fn, ck});
  if (it != memo.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ck * kNumSMs);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ck;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  DPG_CUDA(cudaOccupancyMaxActiveClusters(&n, fn, &cfg));
  if (n <= 0) raise(DPG_ERR_INTERNAL, "cluster split-K: no cluster of " + std::to_string(ck) + " fits");
  memo[{dev, fn, ck}] = n;
  return n;
}

CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box, const uint32_t* estr, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  cuuint64_t d[5], s[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    es[i] = estr ? estr[i] : 1;
    if (i + 1 < rank) s[i] = strides[i];
  }
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(base), d, s,
                               bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(DPG_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// ---- D[M][N] = A[M][K] B[N][K]^T, all row-major (the core's unit test) ----
template <int BN, int BK, bool BMN = false>
struct Gemm2D {
  static constexpr bool kScaleA = false, kBPreSplit = false, kCtaReduce = false, kBMajorMN = BMN;
  static constexpr int kStaging = 0, kEpiIn = 0;
  CUtensorMap ma, mb;
  float* d;
  int M, N, K;
  __device__ int nkb(int) const { return (K + BK - 1) / BK; }
  __device__ uint32_t stage_bytes() const { return (uint32_t)((BM + BN) * BK * 4); }  // (MN: BN/32 boxes)
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t, uint32_t bar, int mt, int nt, int) const {
    tma2(sa, &ma, bar, kb * BK, mt * BM);
    if (BMN) {  // B^T [K][N]: one [BK][32] box per 32-wide N chunk
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tma2(sb + c * (BK * 128), &mb, bar, nt * BN + 32 * c, kb * BK);
    } else {
      tma2(sb, &mb, bar, kb * BK, nt * BN);
    }
  }
  __device__ float scale(int, int, int, int) const { return 1.f; }
  __device__ int a_rows() const { return BM; }
  __device__ bool has_epi_in() const { return false; }
  __device__ uint32_t epi_in_bytes() const { return 0; }
  __device__ void epi_load(int, int, int, int, uint32_t, uint32_t) const {}
  __device__ uint64_t pre_epilogue(int, int, int, int) const { return 0; }
  static constexpr bool kEpiConst = false;
  __device__ void epi_const(int, int, int, int, float*) const {}
  __device__ void epilogue(int mt, int nt, int, int row, int c0, const float (&v)[16], double&, uint8_t*,
                           const uint8_t*, uint64_t, const float*) const {
    const int m = mt * BM + row;
    if (m >= M) return;
    const int n0 = nt * BN + c0;
    if (N % 4 == 0 && n0 + 16 <= N) {  // 16-byte stores
      float4* dp = reinterpret_cast<float4*>(d + (int64_t)m * N + n0);
#pragma unroll
      for (int q = 0; q < 4; ++q) dp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int n = n0 + j;
      if (n < N) d[(int64_t)m * N + n] = v[j];
    }
  }
  __device__ void epi_store(int, int, int, int, uint32_t) const {}
  __device__ void finish(int, int, int, double) const {}
};

// launch with split-K over clusters of ck CTAs (1, 2 or 4)
template <int BN, int BK, class Pr>
void launch_ck(dpg_ctx* ctx, const Pr& p, dim3 grid, int ck) {
  constexpr int STG = Pr::kStaging, EIN = Pr::kEpiIn, AW = acc_width<Pr, BN>();
  switch (ck) {
    case 4: launch<BN, BK, stages_for<BN, BK, STG, EIN, red_bytes(4), AW>(), Pr, 4>(ctx, p, grid); break;
    case 2: launch<BN, BK, stages_for<BN, BK, STG, EIN, red_bytes(2), AW>(), Pr, 2>(ctx, p, grid); break;
    default: launch<BN, BK, stages_for<BN, BK, STG, EIN, 0, AW>(), Pr, 1>(ctx, p, grid); break;
  }
}

template <int BN, int BK, bool BMN = false>
void gemm2d(dpg_ctx* ctx, const float* a, const float* b, float* d, int M, int N, int K, int ck = 1) {
  const uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, db[2] = {(uint64_t)K, (uint64_t)N};
  const uint64_t sa[1] = {(uint64_t)K * 4}, sb[1] = {(uint64_t)K * 4};
  const uint32_t ba[2] = {BK, BM}, bb[2] = {BK, BN};
  Gemm2D<BN, BK, BMN> p;
  p.ma = make_map(a, 2, da, sa, ba, nullptr, KLay<BK>::TMA_SWIZZLE);
  if (BMN) {  // b holds B^T: [K][N] row-major
    const uint64_t dt[2] = {(uint64_t)N, (uint64_t)K}, st[1] = {(uint64_t)N * 4};
    const uint32_t bt[2] = {32, BK};
    p.mb = make_map(b, 2, dt, st, bt, nullptr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  } else {
    p.mb = make_map(b, 2, db, sb, bb, nullptr, KLay<BK>::TMA_SWIZZLE);
  }
  p.d = d; p.M = M; p.N = N; p.K = K;
  const dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN, 1);
  if constexpr (!BMN && BN <= 64) launch_ck<BN, BK>(ctx, p, grid, ck);
  else launch<BN, BK, stages_for<BN, BK>()>(ctx, p, grid);
}

// =============================================================================================
// Convolution contractions. Activations and highways that feed a TMA operand are kept on the
// device in NHWC ("channels last") beside the reference-layout NCHW buffers: a (tap, channel
// block) of the implicit im2col is then one box — channels innermost (one swizzled 64 / 128 B
// row per output position), output positions walked with the convolution stride as the box's
// traversal stride, padding from the out-of-bounds fill. Weights are re-laid and split once per
// step by tg::prep_weights: wf[hi|lo][o][ki][kj][c] (forward, K = (tap, c)) and
// wd[hi|lo][ki][kj][c][o] (dgrad), TF32-rounded hi and lo parts, loaded as the B operand as is.
// Outputs leave through shared memory as TMA bulk stores (NCHW and NHWC copies of a 16-channel
// chunk per store pair), so the epilogue threads issue no per-element global traffic.
// =============================================================================================

// ---- forward: Y[(n, p), o] = bias[o] + sum_(tap, c) X[n, p @ tap, c] W[o, c, tap] ----
// rows of a tile: spt whole samples (spt P <= 128)
template <int BN, int BK>
struct ConvFwdT {
  static constexpr bool kScaleA = false, kBPreSplit = true, kCtaReduce = false, kBMajorMN = false;
  static constexpr int kStaging = 0, kEpiIn = 0;
  CUtensorMap ma, mb;
  int b, O, P, kw, s, pad, spt, cpt, nk, relu_out;
  uint32_t bytes;
  const float* bias;
  float* y;   // NCHW [b][O][P]
  float* yh;  // NHWC [b][P][O] of the consumer's input (ReLU applied when relu_out) or null
  __device__ int nkb(int) const { return nk; }
  __device__ uint32_t stage_bytes() const { return bytes; }
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t sblo, uint32_t bar, int mt, int nt, int) const {
    const int tap = kb / cpt, cb = kb - tap * cpt;
    const int ki = tap / kw, kj = tap - ki * kw;
    tma4(sa, &ma, bar, cb * BK, kj - pad, ki - pad, mt * spt);
    tma3(sb, &mb, bar, kb * BK, nt * BN, 0);
    tma3(sblo, &mb, bar, kb * BK, nt * BN, 1);
  }
  __device__ float scale(int, int, int, int) const { return 1.f; }
  __device__ int a_rows() const { return BM; }
  __device__ bool has_epi_in() const { return false; }
  __device__ uint32_t epi_in_bytes() const { return 0; }
  __device__ void epi_load(int, int, int, int, uint32_t, uint32_t) const {}
  __device__ uint64_t pre_epilogue(int, int, int, int) const { return 0; }
  // the bias of the tile's BN output channels, loaded while the tile's MMAs run
  static constexpr bool kEpiConst = true;
  __device__ void epi_const(int, int nt, int, int row, float* cst) const {
    if (row < BN) cst[row] = (bias && nt * BN + row < O) ? __ldg(bias + nt * BN + row) : 0.f;
  }
  // direct stores: a warp's rows are consecutive positions, so each NCHW store instruction covers
  // whole 16-byte .. 128-byte position runs, and each thread writes its NHWC row's 16 channels as
  // four 16-byte stores (TMA stores of small-P boxes were request-bound: 16-byte NCHW rows)
  __device__ void epilogue(int mt, int nt, int, int row, int c0, const float (&v)[16], double&, uint8_t*,
                           const uint8_t*, uint64_t, const float* cst) const {
    const int r = row / P, pp = row - r * P;
    const int n = mt * spt + r, o0 = nt * BN + c0;
    if (row >= spt * P || n >= b || o0 >= O) return;  // O % 4 == 0; a chunk may straddle O
    float out[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = v[j] + cst[c0 + j];
    float* yp = y + ((int64_t)n * O + o0) * P + pp;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (o0 + j < O) yp[(int64_t)j * P] = out[j];
    if (yh) {
      float* hp = yh + ((int64_t)n * P + pp) * O + o0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (o0 + 4 * c < O)
          *reinterpret_cast<float4*>(hp + 4 * c) =
              make_float4(relu_if(out[4 * c], relu_out), relu_if(out[4 * c + 1], relu_out),
                          relu_if(out[4 * c + 2], relu_out), relu_if(out[4 * c + 3], relu_out));
    }
  }
  __device__ void epi_store(int, int, int, int, uint32_t) const {}
  __device__ void finish(int, int, int, double) const {}
};

// ---- dgrad: dX[n, c, iy, ix] = sum_(o, tap) dY[n, o, (iy + pad - ki) / s, ...] W[o, c, tap] ----
// one launch slice (z) per stride-parity class (py, px) of input pixels; a class only meets the
// taps ki = (py + pad) mod s (+ s ...), each a unit-stride box of the NHWC highway at offset
// (py + pad - ki) / s. Rows of a tile: spt samples x the class grid (QH x QW, the largest class;
// box rows beyond a smaller class's grid fall outside the tensor and are neither loaded nor
// stored). The ReLU mask of the layer input comes in as a TMA box of the NHWC input copy; the
// NHWC result leaves as a TMA store with the class's stride; the NCHW result is stored directly.
template <int BN, int BK>
struct ConvDgradT {
  static constexpr bool kScaleA = false, kBPreSplit = true, kCtaReduce = false, kBMajorMN = false;
  static constexpr int kStaging = 0, kEpiIn = 0;
  CUtensorMap ma, mb;
  int b, C, H, W, kh, kw, s, pad, QH, QW, spt, ocb;
  uint32_t bytes;
  const float* mask_h;  // NHWC [b][H][W][C] layer input (ReLU mask of the input gradient) or null
  float* dxh;           // NHWC [b][H][W][C] input gradient or null
  float* dx;            // NCHW [b][C][H][W] input gradient or null
  __device__ int first_tap(int ph) const { return (ph + pad) % s; }
  __device__ int taps(int k0, int kdim) const { return k0 < kdim ? (kdim - k0 + s - 1) / s : 0; }
  __device__ int nkb(int z) const {
    const int py = z / s, px = z - py * s;
    return taps(first_tap(py), kh) * taps(first_tap(px), kw) * ocb;
  }
  __device__ uint32_t stage_bytes() const { return bytes; }
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t sblo, uint32_t bar, int mt, int nt, int z) const {
    const int py = z / s, px = z - py * s;
    const int t = kb / ocb, ob = kb - t * ocb;
    const int ky0 = first_tap(py), kx0 = first_tap(px);
    const int nkx = taps(kx0, kw);
    const int ti = t / nkx, tj = t - ti * nkx;
    const int ki = ky0 + ti * s, kj = kx0 + tj * s;
    const int dy = (py + pad - ki) / s, dxo = (px + pad - kj) / s;  // exact (multiples of s)
    tma4(sa, &ma, bar, ob * BK, dxo, dy, mt * spt);
    const int brow = (ki * kw + kj) * C + nt * BN;
    tma3(sb, &mb, bar, ob * BK, brow, 0);
    tma3(sblo, &mb, bar, ob * BK, brow, 1);
  }
  __device__ float scale(int, int, int, int) const { return 1.f; }
  __device__ int a_rows() const { return BM; }
  __device__ bool has_epi_in() const { return false; }
  __device__ uint32_t epi_in_bytes() const { return 0; }
  __device__ void epi_load(int, int, int, int, uint32_t, uint32_t) const {}
  // the input pixel of an epilogue row (false: padding row of the tile)
  __device__ bool pixel(int mt, int z, int row, int64_t& pix, int& n, int& iy, int& ix) const {
    const int q = QH * QW;
    if (row >= spt * q) return false;
    const int r = row / q, rr = row - r * q;
    n = mt * spt + r;
    const int qy = rr / QW, qx = rr - qy * QW;
    const int py = z / s, px = z - py * s;
    iy = s * qy + py;
    ix = s * qx + px;
    if (n >= b || iy >= H || ix >= W) return false;
    pix = ((int64_t)n * H + iy) * W + ix;
    return true;
  }
  static constexpr bool kEpiConst = false;
  __device__ void epi_const(int, int, int, int, float*) const {}
  // ReLU mask of the tile's first 64 channels as bits, from the NHWC input copy (one thread reads
  // its pixel's contiguous channels; the loads overlap the tile's MMAs)
  __device__ uint64_t pre_epilogue(int mt, int nt, int z, int row) const {
    int64_t pix;
    int n, iy, ix;
    if (!mask_h || !pixel(mt, z, row, pix, n, iy, ix)) return 0;
    const float4* src = reinterpret_cast<const float4*>(mask_h + pix * C + nt * BN);
    constexpr int NV = (BN < 64 ? BN : 64) / 4;
    float4 m[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) m[i] = __ldg(src + i);
    uint64_t bits = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      bits |= (uint64_t)((m[i].x > 0.f) | (m[i].y > 0.f) << 1 | (m[i].z > 0.f) << 2 | (m[i].w > 0.f) << 3) << (4 * i);
    return bits;
  }
  __device__ void epilogue(int mt, int nt, int z, int row, int c0, const float (&v)[16], double&, uint8_t*,
                           const uint8_t*, uint64_t pre, const float*) const {
    int64_t pix;
    int n, iy, ix;
    if (!pixel(mt, z, row, pix, n, iy, ix)) return;
    const int cb0 = nt * BN + c0;
    if (cb0 >= C) return;  // C % 16 == 0: a chunk is inside or past the channels
    uint32_t mbits = 0xFFFFu;
    if (mask_h) {
      if (c0 < 64) {
        mbits = (uint32_t)(pre >> c0) & 0xFFFFu;
      } else {
        const float4* src = reinterpret_cast<const float4*>(mask_h + pix * C + cb0);
        mbits = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 m = __ldg(src + c);
          mbits |= ((m.x > 0.f) | (m.y > 0.f) << 1 | (m.z > 0.f) << 2 | (m.w > 0.f) << 3) << (4 * c);
        }
      }
    }
    float out[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = (mbits >> j) & 1u ? v[j] : 0.f;
    if (dxh) {
      float4* d = reinterpret_cast<float4*>(dxh + pix * C + cb0);
#pragma unroll
      for (int c = 0; c < 4; ++c) d[c] = make_float4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]);
    }
    if (!dx) return;  // dx null: the NHWC copy is the only output
#pragma unroll
    for (int j = 0; j < 16; ++j) dx[(((int64_t)n * C + cb0 + j) * H + iy) * W + ix] = out[j];
  }
  __device__ void epi_store(int, int, int, int, uint32_t) const {}
  __device__ void finish(int, int, int, double) const {}
};

// ---- clipped sum of a conv weight (clip_and_sum pass 2 as (s ⊙ B)^T A, optimizer.hpp:99-114):
//   S_z[o][c kk + t] = sum over the split's samples n and positions p of
//                      s_n B[n, o, p] X~[n, p, (t, c)]
// M = output channels: the K-major rows s_n B[n, o, p0 .. p0 + BK) of the NCHW highway are the A
// operand, scaled and split into TMEM by the converters (rows past O written as zeros). N = (tap,
// channel) in tap-major order: per 32-channel chunk of a tap, one NHWC box of the layer input
// (ReLU applied by its producer) lands as an MN-major [BK positions][32 channels] tile (32-byte-atom
// swizzle) — the implicit im2col with no transposition. K = (sample, position) of the split, one
// sample per K block (P % BK == 0). Partials [split][O][(tap, channel)], 16-float row pieces per
// epilogue thread; the split-K reduce combines them in a fixed order and writes the reference's
// k order (clip.cu TapMajorOut). Chains are bounded like the register-gather kernel's
// (<= 512 products per TMEM accumulator).
template <int BN, int BK>
struct ConvCsumT {
  static constexpr bool kScaleA = true, kBPreSplit = false, kCtaReduce = false, kBMajorMN = true;
  static constexpr int kStaging = 0, kEpiIn = 0;
  CUtensorMap ma, mb;
  int b, O, C, khw, kw, s, pad, OW, G, kpb, spl;
  uint32_t bytes;
  const float* svec;
  float* part;  // [splits][O][C khw]
  __device__ int a_rows() const { return O; }
  __device__ int nkb(int z) const {
    const int n0 = z * spl, n1 = min(b, n0 + spl);
    return n1 > n0 ? (n1 - n0) * kpb : 0;
  }
  __device__ uint32_t stage_bytes() const { return bytes; }
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t, uint32_t bar, int, int nt, int z) const {
    const int n = z * spl + kb / kpb, j = kb % kpb;
    tma3(sa, &ma, bar, j * BK, 0, n);  // B[n, 0 .. O, p0 .. p0 + BK)
    const int rows = BK / OW, cpc = C / 32;
#pragma unroll 1
    for (int i = 0; i < BN / 32; ++i) {
      const int tl = i / cpc, cc = i - tl * cpc, t = nt * G + tl;
      const int ki = t / kw, kj = t - ki * kw;
      const int y0 = t < khw ? j * rows * s - pad + ki : -(1 << 20);  // past the taps: zeros
      tma4(sb + i * (BK * 128), &mb, bar, cc * 32, kj - pad, y0, n);
    }
  }
  __device__ float scale(int kb, int, int, int z) const { return __ldg(svec + z * spl + kb / kpb); }
  __device__ bool has_epi_in() const { return false; }
  __device__ uint32_t epi_in_bytes() const { return 0; }
  __device__ void epi_load(int, int, int, int, uint32_t, uint32_t) const {}
  __device__ uint64_t pre_epilogue(int, int, int, int) const { return 0; }
  static constexpr bool kEpiConst = false;
  __device__ void epi_const(int, int, int, int, float*) const {}
  __device__ void epilogue(int, int nt, int z, int row, int c0, const float (&v)[16], double&, uint8_t*,
                           const uint8_t*, uint64_t, const float*) const {
    const int K = C * khw, col = nt * G * C + c0;  // tap-major column: (tap, channel)
    if (row >= O || col >= K) return;
    float4* dst = reinterpret_cast<float4*>(part + ((int64_t)z * O + row) * K + col);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  __device__ void epi_store(int, int, int, int, uint32_t) const {}
  __device__ void finish(int, int, int, double) const {}
};

// ---- per-sample gradient of a 3x3 conv weight with 32 input channels (grad_sample.hpp conv2d
// rule: G_n[o][c kk + t] = sum_p B[n, o, p] X~[n, p, (t, c)], layers.hpp:290-324 k order), its
// squared norm (clip_and_sum pass 1) and the materialised record:
// one sample per tile group — three tiles of three taps x 32 channels (N = 96, MN-major NHWC
// input boxes as in ConvCsumT) and the sample's highway rows as the A operand (M = output
// channels). A CTA keeps the three tiles of a sample (blocked schedule) and stages their
// columns in the reference's k order in shared memory (row pitch K + 1: conflict-free), then
// writes the sample's [O][K] record contiguously; the norm is one partial per tile.
template <int BK>
struct ConvRuleT {
  static constexpr int BN = 96, G = 3, NTN = 3, KK = 9, C = 32, K = C * KK, KP = K + 1, OMAX = 64;
  static constexpr bool kScaleA = false, kBPreSplit = false, kCtaReduce = true, kBMajorMN = true;
  static constexpr int kStaging = 0, kEpiIn = 0;
  static constexpr int kTileStg = OMAX * KP * 4, kTileBlock = NTN;
  CUtensorMap ma, mb;
  int b, O, kw, s, pad, OW, kpb;
  uint32_t bytes;
  float* gw;      // record [b][O][K] or null (norms only)
  double* sq;     // norm partials [NTN][b]
  __device__ int a_rows() const { return O; }
  __device__ int nkb(int) const { return kpb; }
  __device__ uint32_t stage_bytes() const { return bytes; }
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t, uint32_t bar, int, int nt, int n) const {
    tma3(sa, &ma, bar, kb * BK, 0, n);  // B[n, 0 .. O, p0 .. p0 + BK)
    const int rows = BK / OW;
#pragma unroll
    for (int tl = 0; tl < G; ++tl) {
      const int t = nt * G + tl, ki = t / kw, kj = t - ki * kw;
      tma4(sb + tl * (BK * 128), &mb, bar, 0, kj - pad, kb * rows * s - pad + ki, n);
    }
  }
  __device__ float scale(int, int, int, int) const { return 1.f; }
  __device__ bool has_epi_in() const { return false; }
  __device__ uint32_t epi_in_bytes() const { return 0; }
  __device__ void epi_load(int, int, int, int, uint32_t, uint32_t) const {}
  __device__ uint64_t pre_epilogue(int, int, int, int) const { return 0; }
  static constexpr bool kEpiConst = false;
  __device__ void epi_const(int, int, int, int, float*) const {}
  __device__ void epilogue(int, int nt, int, int row, int c0, const float (&v)[16], double& acc, uint8_t* stg,
                           const uint8_t*, uint64_t, const float*) const {
    if (row >= O) return;
    const int t = nt * G + c0 / C, cb = c0 % C;  // a chunk is 16 channels of one tap
    float* dst = reinterpret_cast<float*>(stg) + row * KP + cb * KK + t;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      dst[jj * KK] = v[jj];
      acc += (double)v[jj] * (double)v[jj];
    }
  }
  __device__ void epi_store(int, int, int, int, uint32_t) const {}
  __device__ void finish(int, int nt, int n, double sum) const {
    if (sq) sq[(int64_t)nt * b + n] = sum;
  }
  __device__ void tile_done(int, int nt, int n, int tid, int nthreads, uint8_t* stg) const {
    if (nt != NTN - 1 || !gw) return;
    const float* src = reinterpret_cast<const float*>(stg);
    float4* dst = reinterpret_cast<float4*>(gw + (int64_t)n * O * K);
    for (int i4 = tid; i4 < O * K / 4; i4 += nthreads) {  // K % 4 == 0: a float4 never straddles rows
      const int o = (4 * i4) / K, k = 4 * i4 - o * K;
      const float* s4 = src + o * KP + k;
      dst[i4] = make_float4(s4[0], s4[1], s4[2], s4[3]);
    }
  }
};

// ---- helper kernels ----
// per-step weight layouts of one conv layer, TF32-split: wf[h][o][(ki kw + kj) C + c] and
// wd[h][((ki kw + kj) C + c) O + o], h = 0: rna_tf32(w), h = 1: rna_tf32(w - hi)
__global__ void prep_weights_kernel(TgPrepItems items) {
  pdl_wait();
  const TgPrepItem& it = items.item[blockIdx.y];
  const int K = it.C * it.kh * it.kw, khw = it.kh * it.kw;
  const int64_t n = (int64_t)it.O * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(i / K), k = (int)(i - (int64_t)o * K);
    const int c = k / khw, t = k - c * khw;
    const float v = __ldg(it.w + i);
    const float hi = __uint_as_float(rna_tf32(__float_as_uint(v)));
    const float lo = __uint_as_float(rna_tf32(__float_as_uint(v - hi)));
    if (it.wf) {
      const int64_t d = (int64_t)o * K + t * it.C + c;
      it.wf[d] = hi;
      it.wf[n + d] = lo;
    }
    if (it.wd) {
      const int64_t d = ((int64_t)t * it.C + c) * it.O + o;
      it.wd[d] = hi;
      it.wd[n + d] = lo;
    }
  }
  pdl_trigger();
}

// NCHW [b][C][P] -> NHWC [b][P][C] (optionally ReLU'd), one sample plane per block through smem
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ src, int relu, int C, int P, float* __restrict__ dst) {
  extern __shared__ float tile[];
  pdl_wait();
  const int64_t base = (int64_t)blockIdx.x * C * P;
  for (int i = threadIdx.x; i < C * P; i += blockDim.x) {
    const int c = i / P, p = i - c * P;
    tile[p * (C + 1) + c] = relu_if(__ldg(src + base + i), relu);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C * P; i += blockDim.x) {
    const int p = i / C, c = i - p * C;
    dst[base + i] = tile[p * (C + 1) + c];
  }
  pdl_trigger();
}

// ---- host launchers ----
namespace {
// NHWC [b][H][W][C] tiles: box (bc channels, bw x bh positions walked with stride s, bn samples)
CUtensorMap nhwc_map(const float* base, int b, int H, int W, int C, int bc, int bw, int bh, int bn, int s,
                     CUtensorMapSwizzle swz) {
  const uint64_t dims[4] = {(uint64_t)C, (uint64_t)W, (uint64_t)H, (uint64_t)b};
  const uint64_t str[3] = {(uint64_t)C * 4, (uint64_t)W * C * 4, (uint64_t)H * W * C * 4};
  const uint32_t box[4] = {(uint32_t)bc, (uint32_t)(bw * s), (uint32_t)(bh * s), (uint32_t)bn};
  const uint32_t es[4] = {1, (uint32_t)s, (uint32_t)s, 1};
  return make_map(base, 4, dims, str, box, es, swz);
}
// [2][rows][k] (TF32 hi and lo planes): box (bk, box_rows, 1)
CUtensorMap split_rows_map(const float* base, int64_t rows, int64_t k, int bk, int box_rows, CUtensorMapSwizzle swz) {
  const uint64_t dims[3] = {(uint64_t)k, (uint64_t)rows, 2};
  const uint64_t str[2] = {(uint64_t)k * 4, (uint64_t)(rows * k * 4)};
  const uint32_t box[3] = {(uint32_t)bk, (uint32_t)box_rows, 1};
  return make_map(base, 3, dims, str, box, nullptr, swz);
}
// output columns per tile: the widest of 128 / 64 / 32 that still gives >= one CTA per SM
// Output tile width and cluster split-K of a conv launch with `slices` M tiles (x parity classes)
// and nkb K blocks per tile. Estimated time in K-block units: waves x (K blocks per CTA x the MMA
// cost at that N + the epilogue's chunks), the cluster split adding the partial exchange. A
// persistent CTA runs its tiles back to back, so waves = ceil(tiles / co-resident clusters).
// The cluster split is opt-in (DPG_TG_CK=2 or 4 allows it): measured, it does not pay on the
// CIFAR step (negative results).
void pick_tile(int n, int64_t slices, int nkb, int& bn_out, int& ck_out) {
  static const int ck_max = [] {
    const char* e = std::getenv("DPG_TG_CK");
    return e ? std::max(1, std::min(4, std::atoi(e))) : 1;
  }();
  double best = 1e30;
  bn_out = 32;
  ck_out = 1;
  for (int bn : {128, 64, 32}) {
    if (bn > ((n + 15) / 16) * 16 + 15) continue;
    const int64_t tiles = slices * ((n + bn - 1) / bn);
    for (int ck : {1, 2, 4}) {
      if (ck > ck_max || (ck > 1 && (bn > 64 || nkb < 2 * ck))) continue;
      const int64_t slots = kNumSMs / ck;
      const int64_t waves = (tiles + slots - 1) / slots;
      const double mma = bn <= 64 ? 1.0 : 1.3;
      const double epi = 0.15 * (bn / 16) * (ck > 1 ? 2.0 : 1.0);
      const double t = (double)waves * ((double)((nkb + ck - 1) / ck) * mma + epi);
      if (t < best - 1e-9) {
        best = t;
        bn_out = bn;
        ck_out = ck;
      }
    }
  }
}
template <class F>
void with_bn(int bn, F&& f) {
  switch (bn) {
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 64: f(std::integral_constant<int, 64>{}); break;
    default: f(std::integral_constant<int, 32>{}); break;
  }
}
template <class F>
void with_bk(int bk, F&& f) {
  if (bk == 32) f(std::integral_constant<int, 32>{});
  else f(std::integral_constant<int, 16>{});
}
}  // namespace

bool fwd_nhwc_ok(const ConvGeom& g) {
  return g.ic % 16 == 0 && g.oc % 4 == 0 && g.P() <= BM && g.P() % 4 == 0 && g.ow * g.stride <= 256 &&
         g.oh * g.stride <= 256;
}
bool dgrad_nhwc_ok(const ConvGeom& g) {
  const int64_t qh = (g.h + g.stride - 1) / g.stride, qw = (g.w + g.stride - 1) / g.stride;
  return g.oc % 16 == 0 && g.ic % 16 == 0 && qh * qw <= BM && qw * g.stride <= 256 && qh * g.stride <= 256;
}

void conv_fwd_nhwc(dpg_ctx* ctx, const float* xh, const float* wf, const float* bias, const ConvGeom& g, float* y,
                   float* yh, int relu_out) {
  const int b = (int)g.b, P = (int)g.P();
  const int spt = BM / P;
  const int64_t mtiles = (b + spt - 1) / spt;
  const int bk = g.ic % 32 == 0 ? 32 : 16;
  int bn, ck;
  pick_tile((int)g.oc, mtiles, (int)(g.kh * g.kw * (g.ic / bk)), bn, ck);
  with_bk(bk, [&](auto BKc) {
    constexpr int BK = decltype(BKc)::value;
    with_bn(bn, [&](auto BNc) {
      constexpr int BN = decltype(BNc)::value;
      using Pr = ConvFwdT<BN, BK>;
      Pr p;
      p.ma = nhwc_map(xh, b, (int)g.h, (int)g.w, (int)g.ic, BK, (int)g.ow, (int)g.oh, spt, (int)g.stride,
                      KLay<BK>::TMA_SWIZZLE);
      p.mb = split_rows_map(wf, g.oc, g.K(), BK, BN, KLay<BK>::TMA_SWIZZLE);
      p.y = y;
      p.yh = yh;
      p.b = b; p.O = (int)g.oc; p.P = P; p.kw = (int)g.kw; p.s = (int)g.stride; p.pad = (int)g.pad;
      p.spt = spt; p.cpt = (int)g.ic / BK; p.nk = (int)(g.kh * g.kw) * p.cpt; p.relu_out = relu_out;
      p.bytes = (uint32_t)((spt * P + 2 * BN) * BK * 4);
      p.bias = bias;
      const dim3 grid((unsigned)mtiles, (unsigned)((g.oc + BN - 1) / BN), 1);
      if constexpr (BN <= 64) launch_ck<BN, BK>(ctx, p, grid, ck);
      else launch<BN, BK, stages_for<BN, BK, Pr::kStaging, Pr::kEpiIn, 0, acc_width<Pr, BN>()>()>(ctx, p, grid);
    });
  });
}

void conv_dgrad_nhwc(dpg_ctx* ctx, const float* hh, const float* wd, const ConvGeom& g, const float* mask_h,
                     float* dx, float* dxh) {
  const int b = (int)g.b, s = (int)g.stride;
  const int QH = (int)((g.h + s - 1) / s), QW = (int)((g.w + s - 1) / s);
  const int spt = BM / (QH * QW);
  const int64_t mtiles = (b + spt - 1) / spt;
  const int bk = g.oc % 32 == 0 ? 32 : 16;
  int bn, ck;  // K blocks per tile: at most ceil(kh / s) ceil(kw / s) taps x the channel blocks
  pick_tile((int)g.ic, mtiles * s * s, (int)(((g.kh + s - 1) / s) * ((g.kw + s - 1) / s) * (g.oc / bk)), bn, ck);
  with_bk(bk, [&](auto BKc) {
    constexpr int BK = decltype(BKc)::value;
    with_bn(bn, [&](auto BNc) {
      constexpr int BN = decltype(BNc)::value;
      using Pr = ConvDgradT<BN, BK>;
      Pr p;
      // unit-stride boxes over the highway (NHWC [b][OH][OW][O])
      p.ma = nhwc_map(hh, b, (int)g.oh, (int)g.ow, (int)g.oc, BK, QW, QH, spt, 1, KLay<BK>::TMA_SWIZZLE);
      p.mb = split_rows_map(wd, g.kh * g.kw * g.ic, g.oc, BK, BN, KLay<BK>::TMA_SWIZZLE);
      p.mask_h = mask_h;
      p.dxh = dxh;
      p.b = b; p.C = (int)g.ic; p.H = (int)g.h; p.W = (int)g.w; p.kh = (int)g.kh; p.kw = (int)g.kw;
      p.s = s; p.pad = (int)g.pad; p.QH = QH; p.QW = QW; p.spt = spt; p.ocb = (int)g.oc / BK;
      p.bytes = (uint32_t)((spt * QH * QW + 2 * BN) * BK * 4);
      p.dx = dx;
      const dim3 grid((unsigned)mtiles, (unsigned)((g.ic + BN - 1) / BN), (unsigned)(s * s));
      if constexpr (BN <= 64) launch_ck<BN, BK>(ctx, p, grid, ck);
      else launch<BN, BK, stages_for<BN, BK, Pr::kStaging, Pr::kEpiIn, 0, acc_width<Pr, BN>()>()>(ctx, p, grid);
    });
  });
}

// ---- per-sample gradient + norm of a conv weight on the core ----
bool rule_nhwc_ok(const ConvGeom& g) {
  const int64_t P = g.P();
  return g.ic == 32 && g.kh == 3 && g.kw == 3 && g.oc <= 64 && P % 32 == 0 && 32 % g.ow == 0 &&
         g.ow * g.stride <= 256 && (32 / g.ow) * g.stride <= 256;
}

void conv_rule_nhwc(dpg_ctx* ctx, const float* xh, const float* hw, const ConvGeom& g, float* gw, double* sq) {
  constexpr int BK = 32;
  using Pr = ConvRuleT<BK>;
  const int b = (int)g.b, P = (int)g.P();
  Pr p;
  {  // A: highway NCHW [b][O][P], K-major rows of BK positions
    const uint64_t dims[3] = {(uint64_t)P, (uint64_t)g.oc, (uint64_t)b};
    const uint64_t str[2] = {(uint64_t)P * 4, (uint64_t)(g.oc * P * 4)};
    const uint32_t box[3] = {(uint32_t)BK, (uint32_t)g.oc, 1};
    p.ma = make_map(hw, 3, dims, str, box, nullptr, KLay<BK>::TMA_SWIZZLE);
  }
  p.mb = nhwc_map(xh, b, (int)g.h, (int)g.w, 32, 32, (int)g.ow, BK / (int)g.ow, 1, (int)g.stride,
                  CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  p.b = b; p.O = (int)g.oc; p.kw = (int)g.kw; p.s = (int)g.stride; p.pad = (int)g.pad; p.OW = (int)g.ow;
  p.kpb = P / BK;
  p.bytes = (uint32_t)(((int)g.oc + Pr::BN) * BK * 4);
  p.gw = gw; p.sq = sq;
  launch<Pr::BN, BK, stages_for<Pr::BN, BK, 0, 0, Pr::kTileStg>()>(ctx, p, dim3(1, Pr::NTN, (unsigned)b));
}

// ---- clipped sum of a conv weight on the core ----
bool csum_nhwc_ok(const ConvGeom& g) {
  const int64_t P = g.P();
  const int bk = P % 32 == 0 ? 32 : 16;
  return (g.ic == 32 || g.ic == 64) && g.oc <= 128 && P % bk == 0 && bk % g.ow == 0 &&
         g.ow * g.stride <= 256 && (bk / g.ow) * g.stride <= 256 && g.kh * g.kw <= 64;
}
int csum_nhwc_splits(const ConvGeom& g) {
  // chains of <= 512 products per TMEM accumulator (tc_conv.cu kCsumChain), and >= one tile per SM
  const int64_t P = g.P();
  const int G = 3, ntn = (int)((g.kh * g.kw + G - 1) / G);
  const int64_t spl_chain = std::max<int64_t>(1, 512 / P);
  // about two tiles per SM: the persistent CTAs overlap one tile's epilogue with the next's loads
  const int64_t want = (2 * kNumSMs + ntn - 1) / ntn;
  int64_t spl = std::min<int64_t>(spl_chain, std::max<int64_t>(1, (g.b + want - 1) / want));
  if (const char* e = std::getenv("DPG_TG_CSUM_SPL")) spl = std::min<int64_t>(spl_chain, std::max(1, std::atoi(e)));
  return (int)((g.b + spl - 1) / spl);
}

void conv_csum_nhwc(dpg_ctx* ctx, const float* xh, const float* hw, const float* scale, const ConvGeom& g,
                    float* part, int splits) {
  const int b = (int)g.b, P = (int)g.P(), C = (int)g.ic, khw = (int)(g.kh * g.kw);
  const int bk = P % 32 == 0 ? 32 : 16;
  constexpr int G = 3;  // taps per N tile
  auto go = [&](auto BNc, auto BKc) {
    constexpr int BN = decltype(BNc)::value, BK = decltype(BKc)::value;
    using Pr = ConvCsumT<BN, BK>;
    Pr p;
    {  // A: highway NCHW [b][O][P], K-major rows of BK positions
      const uint64_t dims[3] = {(uint64_t)P, (uint64_t)g.oc, (uint64_t)b};
      const uint64_t str[2] = {(uint64_t)P * 4, (uint64_t)(g.oc * P * 4)};
      const uint32_t box[3] = {(uint32_t)BK, (uint32_t)g.oc, 1};
      p.ma = make_map(hw, 3, dims, str, box, nullptr, KLay<BK>::TMA_SWIZZLE);
    }
    // B: the layer input NHWC, 32-channel boxes of BK / OW output rows walked with the stride
    p.mb = nhwc_map(xh, b, (int)g.h, (int)g.w, C, 32, (int)g.ow, BK / (int)g.ow, 1, (int)g.stride,
                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    p.b = b; p.O = (int)g.oc; p.C = C; p.khw = khw; p.kw = (int)g.kw; p.s = (int)g.stride; p.pad = (int)g.pad;
    p.OW = (int)g.ow; p.G = G; p.kpb = P / BK; p.spl = (b + splits - 1) / splits;
    p.bytes = (uint32_t)(((int)g.oc + BN) * BK * 4);
    p.svec = scale; p.part = part;
    launch<BN, BK, stages_for<BN, BK>()>(ctx, p, dim3(1, (unsigned)((khw + G - 1) / G), (unsigned)splits));
  };
  if (C == 32) {
    if (bk == 32) go(std::integral_constant<int, 96>{}, std::integral_constant<int, 32>{});
    else go(std::integral_constant<int, 96>{}, std::integral_constant<int, 16>{});
  } else {
    if (bk == 32) go(std::integral_constant<int, 192>{}, std::integral_constant<int, 32>{});
    else go(std::integral_constant<int, 192>{}, std::integral_constant<int, 16>{});
  }
}

void prep_weights(dpg_ctx* ctx, const TgPrepItems& items) {
  if (items.count == 0) return;
  ::dpg::launch_pdl(prep_weights_kernel, dim3(2 * kNumSMs / items.count + 1, (unsigned)items.count), 256, 0,
                    ctx->stream, items);
  DPG_LAUNCH_CHECK(ctx);
}

void nchw_to_nhwc(dpg_ctx* ctx, const float* src, int relu, int64_t b, int64_t C, int64_t P, float* dst) {
  const int smem = (int)(sizeof(float) * P * (C + 1));
  if (smem > 96 * 1024) raise(DPG_ERR_DIMENSION, "nchw_to_nhwc: sample plane too large");
  ensure_smem_attr(reinterpret_cast<const void*>(nchw_to_nhwc_kernel), smem);
  ::dpg::launch_pdl(nchw_to_nhwc_kernel, (unsigned)b, 256, smem, ctx->stream, src, relu, (int)C, (int)P, dst);
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace tg
}  // namespace dpg

#ifdef DPG_TG_TRACE
// trace builds only (tools/tg_trace_step.py): read the traced launch's timeline
extern "C" __attribute__((visibility("default"))) void dpg_tg_trace_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, dpg::tg::g_tg_trace, sizeof(unsigned long long) * 10 * 256);
}
#endif

using dpg::guard;
using dpg::raise;

dpg_status dpg_tg_gemm_selftest_split(dpg_ctx* ctx, const float* a, const float* b, float* d, int64_t m,
                                      int64_t n, int64_t k, int bn, int ck) {
  return guard(ctx, [&] {
    if (!ctx) raise(DPG_ERR_PARAMETER, "null context");
    if (m <= 0 || n <= 0 || k <= 0 || (k * 4) % 16 != 0 || m >= (1 << 30) || n >= (1 << 30) || k >= (1 << 30))
      raise(DPG_ERR_DIMENSION, "tg_gemm_selftest_split: extents must be positive, K a multiple of 4");
    if (ck != 1 && ck != 2 && ck != 4) raise(DPG_ERR_PARAMETER, "tg_gemm_selftest_split: ck must be 1, 2 or 4");
    switch (bn) {
      case 32: dpg::tg::gemm2d<32, 32>(ctx, a, b, d, (int)m, (int)n, (int)k, ck); break;
      case 64: dpg::tg::gemm2d<64, 32>(ctx, a, b, d, (int)m, (int)n, (int)k, ck); break;
      default: raise(DPG_ERR_PARAMETER, "tg_gemm_selftest_split: bn must be 32 or 64");
    }
  });
}

dpg_status dpg_tg_gemm_selftest(dpg_ctx* ctx, const float* a, const float* b, float* d, int64_t m, int64_t n,
                                int64_t k, int bn, int bk) {
  return guard(ctx, [&] {
    if (!ctx) raise(DPG_ERR_PARAMETER, "null context");
    if (m <= 0 || n <= 0 || k <= 0 || (k * 4) % 16 != 0 || m >= (1 << 30) || n >= (1 << 30) || k >= (1 << 30))
      raise(DPG_ERR_DIMENSION, "tg_gemm_selftest: extents must be positive, K a multiple of 4");
    const int M = (int)m, N = (int)n, K = (int)k;
    if (bk == -32) {  // B given transposed ([K][N] row-major): the MN-major B path
      if (n % 4 != 0) raise(DPG_ERR_DIMENSION, "tg_gemm_selftest: MN-major B needs N a multiple of 4");
      switch (bn) {
        case 32: dpg::tg::gemm2d<32, 32, true>(ctx, a, b, d, M, N, K); break;
        case 64: dpg::tg::gemm2d<64, 32, true>(ctx, a, b, d, M, N, K); break;
        case 96: dpg::tg::gemm2d<96, 32, true>(ctx, a, b, d, M, N, K); break;
        case 192: dpg::tg::gemm2d<192, 32, true>(ctx, a, b, d, M, N, K); break;
        default: raise(DPG_ERR_PARAMETER, "tg_gemm_selftest: bn must be 32, 64, 96 or 192 with bk -32");
      }
    } else if (bk == 32) {
      switch (bn) {
        case 32: dpg::tg::gemm2d<32, 32>(ctx, a, b, d, M, N, K); break;
        case 64: dpg::tg::gemm2d<64, 32>(ctx, a, b, d, M, N, K); break;
        case 128: dpg::tg::gemm2d<128, 32>(ctx, a, b, d, M, N, K); break;
        default: raise(DPG_ERR_PARAMETER, "tg_gemm_selftest: bn must be 32, 64 or 128");
      }
    } else if (bk == 16) {
      switch (bn) {
        case 32: dpg::tg::gemm2d<32, 16>(ctx, a, b, d, M, N, K); break;
        case 64: dpg::tg::gemm2d<64, 16>(ctx, a, b, d, M, N, K); break;
        default: raise(DPG_ERR_PARAMETER, "tg_gemm_selftest: bn must be 32 or 64 with bk 16");
      }
    } else {
      raise(DPG_ERR_PARAMETER, "tg_gemm_selftest: bk must be 16 or 32");
    }
  });
}
