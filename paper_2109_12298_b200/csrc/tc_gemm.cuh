// tc_gemm.cuh — tcgen05 (5th-gen tensor core) implicit GEMM, 3xTF32 fp32-faithful.
//
//   C[z][m][n] = sum_k A(z, m, k) * B(z, n, k)         (both operands K-major)
//
// Operands are gathered by all threads of the CTA through a problem-specific stage loader (the
// implicit im2col of the conv contractions lives there, driven by per-CTA index tables in shared
// memory), split into a TF32 "hi" part and the TF32-rounded remainder "lo" (split_tf32), and stored
// into shared memory in the canonical swizzled K-major UMMA layout (8-row atoms of 64 B or 128 B
// rows, 1024 B aligned). One thread issues tcgen05.mma.cta_group::1.kind::tf32 with the accumulator in
// tensor memory: acc += A_lo B_hi + A_hi B_lo + A_hi B_hi per K=8 slice (3xTF32). Stages are
// double buffered: the MMAs of stage s run asynchronously while the threads gather stage s+1;
// tcgen05.commit arrives on the stage's mbarrier to release the buffer.
//
// Operands for stage s+2 are fetched into registers while stage s is stored and its MMAs run.
//
// Epilogue: tcgen05.ld; warp w owns TMEM lanes [32 (w % 4), +32) (= tile rows) and the column
// half w / 4; each thread hands its row's values to Prob::epilogue_row.
//
// Split-K: blockIdx.z = z * ksplit + split; split s covers K stages [s * nk / ksplit,
// (s + 1) * nk / ksplit) and the Prob writes a partial that a fixed-order reduce combines.
//
// Tile: BM = 128 rows (UMMA M), BN in {16, 32, 64, 128} columns (UMMA N), BK = 16 fp32 (one
// 64 B swizzle row; 32 with DPG_TC_BK=32) per stage; 256 threads.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "dpg_device.cuh"

namespace dpg {
namespace tc {

constexpr int BM = 128;
// every problem carries its rows per CTA tile (<= BM; set by launch_tc)
struct TileRows {
  int mstep = BM;
};
// K per stage: 16 fp32 = one 64 B swizzle row (SWIZZLE_64B) keeps a stage at 24 KB for BN = 64, so
// three CTAs fit an SM (shared memory and registers); DPG_TC_BK=32 selects 128 B rows (SWIZZLE_128B).
#ifndef DPG_TC_BK
#define DPG_TC_BK 16
#endif
#ifndef DPG_TC_EXP
#define DPG_TC_EXP 0  // timing experiments only (results wrong): 1 = skip gathers, 2 = skip stores, 4 = skip MMAs
#endif
#ifndef DPG_TC_MINB
#define DPG_TC_MINB 4  // resident CTAs per SM the 16-wide-K kernel is register-budgeted for (64 regs)
#endif
constexpr int BK = DPG_TC_BK;
static_assert(BK == 16 || BK == 32, "BK: one 64 B or 128 B swizzle row");
constexpr int kQuadsPerRow = BK / 4;                 // 16 B chunks per K-major row
constexpr int kRowBytes = BK * 4;                    // 64 or 128
constexpr int kAtomBytes = 8 * kRowBytes;            // 8-row swizzle atom: 512 or 1024
constexpr int kAQ = BM * kQuadsPerRow / 256;         // A quads per thread per stage: 2 or 4
constexpr uint64_t kLayoutType = BK == 32 ? 2 : 4;   // UMMA layout: SWIZZLE_128B / SWIZZLE_64B
constexpr int kMinBlocks = BK == 32 ? 2 : DPG_TC_MINB;         // resident CTAs per SM the kernel is built for
constexpr int kThreads = 256;
#ifndef DPG_TC_TRUNC
// 3xTF32 with a truncated hi part: step -0.9 %, but biased. With hi = trunc(x), lo has the sign
// of x and |lo| < 2^-10 |x|, so the dropped lo*lo product (up to 2^-20 |x w|) shrinks every
// product toward zero; a long cancelling sum accumulates that linearly (b = 4096 conv2 clipped
// sum: 1.28e-5 max-scaled vs fp64, against the fp32 reference's own 2.2e-6). Rounded parts
// leave a zero-mean lo*lo of <= 2^-22 |x w|: the default.
#define DPG_TC_TRUNC 0
#endif
#ifndef DPG_TC_STAGES
#define DPG_TC_STAGES 2
#endif
constexpr int kStages = DPG_TC_STAGES;  // shared-memory stage ring

// ---- integer division by a runtime constant (multiply-high), valid for n < 2^31 ----
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (div <= 1) {
      d = 1;
      return;
    }
    uint32_t l = 0;
    while ((1u << l) < div) ++l;  // ceil(log2 div)
    s = 31 + l;
    m = (uint32_t)(((1ull << s) + div - 1) / div);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return d == 1 ? n : (uint32_t)(((uint64_t)n * m) >> s);
  }
  __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

// ---- PTX wrappers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Swizzled K-major shared memory descriptor (tcgen05 matrix descriptor, sm_100 version 1):
// start >> 4 | LBO 16 B >> 4 | SBO = one 8-row atom >> 4 | version 1 | layout (SWIZZLE_64B/128B)
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(kAtomBytes >> 4) << 32) |
         ((uint64_t)1 << 46) | (kLayoutType << 61);
}

// Instruction descriptor kind::tf32: D f32, A/B tf32, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 16 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// byte offset of (row, 16 B chunk q) in a swizzled K-major tile: the 16 B chunk index is XORed
// with address bits [7, 7 + log2(chunks per row)) — (row & 7) for 128 B rows, (row >> 1) & 3 for
// 64 B rows (CuTe Swizzle<3,4,3> / Swizzle<2,4,3>)
__device__ __forceinline__ uint32_t sw_off(int row, int q) {
  const int x = BK == 32 ? (row & 7) : ((row >> 1) & 3);
  return (uint32_t)((row >> 3) * kAtomBytes + (row & 7) * kRowBytes + ((q ^ x) << 4));
}

// 3xTF32 split of a finite fp32 value. DPG_TC_TRUNC=1: hi = x as stored, which the
// tensor core reads as trunc_tf32(x) (top 19 bits), lo = x - trunc_tf32(x), exact in fp32 and
// itself truncated by the MMA: |error| <= 2^-21 |x| per operand, two ops. DPG_TC_TRUNC=0 (default): both
// parts rounded to nearest (ties away, as cvt.rna) by integer add + mask, |error| <= 2^-22 |x|,
// five ops. No special-case branches either way; a non-finite x still gives a non-finite
// product, which the clip-factor check reports.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
#if DPG_TC_TRUNC
  // the MMA reads the top 19 bits of each 32-bit operand: store x itself as "hi" and the exact
  // remainder x - trunc_tf32(x) as "lo" (two ops)
  hi = __float_as_uint(x);
  lo = __float_as_uint(x - __uint_as_float(hi & 0xffffe000u));
#else
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = (__float_as_uint(x - __uint_as_float(hi)) + 0x1000u) & 0xffffe000u;
#endif
}

// Store 4 values (k .. k+3 of one row) as hi / lo TF32 into the swizzled stage buffers.
__device__ __forceinline__ void put4(uint8_t* hi, uint8_t* lo, int row, int q, float a, float b,
                                     float c, float d) {
  const uint32_t off = sw_off(row, q);
  uint4 h, l;
  split_tf32(a, h.x, l.x);
  split_tf32(b, h.y, l.y);
  split_tf32(c, h.z, l.z);
  split_tf32(d, h.w, l.w);
  *reinterpret_cast<uint4*>(hi + off) = h;
  *reinterpret_cast<uint4*>(lo + off) = l;
}
__device__ __forceinline__ void put4(uint8_t* hi, uint8_t* lo, int row, int q, float4 v) {
  put4(hi, lo, row, q, v.x, v.y, v.z, v.w);
}

template <int BN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 4;  // 8 or 16 KB
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int FIXED = kStages * STAGE + 64;
};

template <int BN>
constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
}

// Stage buffers
struct StageBufsT {
  uint8_t* a_hi;
  uint8_t* a_lo;
  uint8_t* b_hi;
  uint8_t* b_lo;
};

// Operand registers of one stage: each thread fetches 4 quads of A (16 floats) and BQ quads of B
// for the NEXT stage while the current one is converted, stored and consumed by the MMA, so
// ~16 + 4 BQ independent loads per thread stay in flight.
//
// Thread -> (row, quad) maps (i = 0..kAQ-1 for A, i = 0..BQ-1 for B; Q = quads per row):
//   A row-major  (kAQuadMajor = false): row = tid & 127, quad = (tid >> 7) + 2 i
//                 — a warp covers 32 rows at one k (coalesced when rows are contiguous)
//   A quad-major (kAQuadMajor = true):  idx = tid + 256 i, row = idx / Q, quad = idx % Q
//                 — a warp covers 32 / Q rows x Q quads (coalesced when K is contiguous)
//   B: idx = tid + 256 i, row = idx / Q, quad = idx % Q (kBQuadMajor) or row = idx % BN,
//      quad = idx / BN
template <int BN>
struct Frag {
  static constexpr int BQ = (BN * kQuadsPerRow + kThreads - 1) / kThreads;
};

__device__ __forceinline__ void a_map(bool quad_major, int tid, int i, int& row, int& q) {
  if (quad_major) {
    const int idx = tid + kThreads * i;
    row = idx / kQuadsPerRow;
    q = idx % kQuadsPerRow;
  } else {
    row = tid & 127;
    q = (tid >> 7) + 2 * i;
  }
}
template <int BN>
__device__ __forceinline__ bool b_map(bool quad_major, int tid, int i, int& row, int& q) {
  const int idx = tid + kThreads * i;
  if (quad_major) {
    row = idx / kQuadsPerRow;
    q = idx % kQuadsPerRow;
  } else {
    row = idx % BN;
    q = idx / BN;
  }
  return idx < BN * kQuadsPerRow;
}

// Prob interface:
//   int64_t M, N, K; int ksplit; int scratch;          max sizes, split-K factor, scratch bytes
//   int64_t mdim(int z), kdim(int z) const;             per-batch M and K (<= M, K)
//   static constexpr bool kAQuadMajor, kBQuadMajor, kCtaReduce;
//   void setup(int z, int64_t m0, int64_t n0, uint8_t* scratch, int tid) const;   once per CTA
//   float4 a_quad(int z, int64_t m0, int row, int64_t k, const uint8_t* scratch) const;
//   float4 b_quad(int z, int64_t n0, int row, int64_t k, const uint8_t* scratch) const;
//        (4 consecutive k starting at k, raw loads; zero outside the problem)
//   float4 a_fix(...same..., float4 v) const; float4 b_fix(...same..., float4 v) const;
//        (applied when the stage is stored: ReLU of a folded activation, clip scale, ...)
//   void epilogue_row(int z, int split, int64_t m, int64_t n, const float* v, int nv, double& sq);
//   void epilogue_cta(int z, int split, int tile_mn, double sq) const;   (tile_mn = n tile * m tiles + m tile)
// Rows of the tile beyond the problem (row >= mrows / nrows: padding of a small M or N up to the
// UMMA shape) are neither gathered nor stored: their shared-memory rows keep stale values, which
// only reach accumulator rows / columns that the epilogue never writes.
template <int BN, class Prob>
__device__ __forceinline__ void fetch(const Prob& p, int z, int64_t m0, int64_t n0, int64_t k0,
                                      const uint8_t* scratch, int tid, int mrows, int nrows,
                                      float4 (&ra)[kAQ], float4 (&rb)[Frag<BN>::BQ]) {
#pragma unroll
  for (int i = 0; i < kAQ; ++i) {
    int row, q;
    a_map(Prob::kAQuadMajor, tid, i, row, q);
    if (row < mrows) ra[i] = p.a_quad(z, m0, row, k0 + 4 * q, scratch);
  }
#pragma unroll
  for (int i = 0; i < Frag<BN>::BQ; ++i) {
    int row, q;
    if (b_map<BN>(Prob::kBQuadMajor, tid, i, row, q) && row < nrows)
      rb[i] = p.b_quad(z, n0, row, k0 + 4 * q, scratch);
  }
}

template <int BN, class Prob>
__device__ __forceinline__ void stash(const Prob& p, int z, int64_t m0, int64_t n0, int64_t k0,
                                      const uint8_t* scratch, int tid, int mrows, int nrows,
                                      const StageBufsT& sb, const float4 (&ra)[kAQ],
                                      const float4 (&rb)[Frag<BN>::BQ]) {
#pragma unroll
  for (int i = 0; i < kAQ; ++i) {
    int row, q;
    a_map(Prob::kAQuadMajor, tid, i, row, q);
    if (row < mrows) put4(sb.a_hi, sb.a_lo, row, q, p.a_fix(z, m0, row, k0 + 4 * q, scratch, ra[i]));
  }
#pragma unroll
  for (int i = 0; i < Frag<BN>::BQ; ++i) {
    int row, q;
    if (b_map<BN>(Prob::kBQuadMajor, tid, i, row, q) && row < nrows)
      put4(sb.b_hi, sb.b_lo, row, q, p.b_fix(z, n0, row, k0 + 4 * q, scratch, rb[i]));
  }
}

template <int BN, class Prob>
__global__ void __launch_bounds__(kThreads, kMinBlocks) tc_gemm_kernel(const Prob p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024 B alignment by pointer arithmetic on the __shared__ array, so the compiler keeps the
  // shared address space (LDS / STS, not generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  using S = Smem<BN>;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * S::STAGE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kStages);
  uint8_t* scratch = smem + S::FIXED;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int z = blockIdx.z / p.ksplit, split = blockIdx.z % p.ksplit;
  const int64_t m0 = (int64_t)blockIdx.x * p.mstep, n0 = (int64_t)blockIdx.y * BN;
  constexpr uint32_t kCols = tmem_cols<BN>();
  const int64_t Mz = p.mdim(z), Kz = p.kdim(z);
  if (m0 >= Mz) return;  // ragged batches (e.g. dgrad parity classes): whole CTA idle

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  p.setup(z, m0, n0, scratch, tid);  // index tables: geometry only, no upstream data
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // TMEM allocation, barrier init and the tables above overlap the previous kernel's tail
  const uint32_t tmem = *tmem_slot;

  const int nk_all = (int)((Kz + BK - 1) / BK);
  const int ks0 = (int)((int64_t)split * nk_all / p.ksplit);
  const int ks1 = (int)((int64_t)(split + 1) * nk_all / p.ksplit);
  const int nk = ks1 - ks0;
  constexpr uint32_t idesc = idesc_tf32(BN);
  // Two register sets: the operands of stage i + 2 are requested while stage i is stored, so each
  // gather has a full stage period (store + barrier + MMA issue of the previous stage) to land.
  float4 ra0[kAQ], rb0[Frag<BN>::BQ], ra1[kAQ], rb1[Frag<BN>::BQ];
  const int mrows = (int)std::min<int64_t>(p.mstep, Mz - m0);
  const int nrows = (int)std::min<int64_t>(BN, p.N - n0);
  if (nk > 0) fetch<BN>(p, z, m0, n0, (int64_t)ks0 * BK, scratch, tid, mrows, nrows, ra0, rb0);
  if (nk > 1) fetch<BN>(p, z, m0, n0, (int64_t)(ks0 + 1) * BK, scratch, tid, mrows, nrows, ra1, rb1);
  auto stage = [&](int i, float4 (&ra)[kAQ], float4 (&rb)[Frag<BN>::BQ]) {
    const int s = i % kStages;
    uint8_t* st = smem + s * S::STAGE;
    const StageBufsT sb{st, st + S::A_BYTES, st + 2 * S::A_BYTES, st + 2 * S::A_BYTES + S::B_BYTES};
    if (i >= kStages) mbar_wait(&bars[s], ((i / kStages) - 1) & 1);
#if DPG_TC_EXP & 2
    if (i < 0)
#endif
    stash<BN, Prob>(p, z, m0, n0, (int64_t)(ks0 + i) * BK, scratch, tid, mrows, nrows, sb, ra, rb);
#if DPG_TC_EXP & 1
    if (i < 0)
#endif
    if (i + 2 < nk) fetch<BN>(p, z, m0, n0, (int64_t)(ks0 + i + 2) * BK, scratch, tid, mrows, nrows, ra, rb);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa_hi = smem_u32(sb.a_hi), sa_lo = smem_u32(sb.a_lo);
      const uint32_t sb_hi = smem_u32(sb.b_hi), sb_lo = smem_u32(sb.b_lo);
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        if (DPG_TC_EXP & 4) break;
        const uint32_t off = kk * 32;  // 8 tf32 = 32 B along the swizzled row
        const uint32_t acc0 = (i > 0 || kk > 0) ? 1u : 0u;
        mma_tf32(tmem, sw_desc(sa_lo + off), sw_desc(sb_hi + off), idesc, acc0);
        mma_tf32(tmem, sw_desc(sa_hi + off), sw_desc(sb_lo + off), idesc, 1u);
        mma_tf32(tmem, sw_desc(sa_hi + off), sw_desc(sb_hi + off), idesc, 1u);
      }
      mma_commit(&bars[s]);
    }
  };
#pragma unroll 1
  for (int i = 0; i < nk; i += 2) {
    stage(i, ra0, rb0);
    if (i + 1 < nk) stage(i + 1, ra1, rb1);
  }
  if (nk > 0) mbar_wait(&bars[(nk - 1) % kStages], ((nk - 1) / kStages) & 1);
  tc_fence_after();
  // the main loop is done: the next kernel may launch during the epilogues
  pdl_trigger();

  // epilogue: warp w -> TMEM lanes [32 (w % 4), +32), columns [(w / 4) BN / 2, +BN / 2)
  const int lane_base = 32 * (warp & 3);
  const int64_t m = m0 + lane_base + (tid & 31);
  const bool row_ok = lane_base + (tid & 31) < mrows;
  constexpr int HALF = BN / 2 >= 16 ? BN / 2 : 16;
  const int c_begin = (warp >> 2) * HALF;
  double sq = 0.0;
  float v[16];
  if (c_begin < BN) {
#pragma unroll 1
    for (int c0 = c_begin; c0 < c_begin + HALF && c0 < BN; c0 += 16) {
      if (nk > 0) {
        tmem_ld16(tmem + ((uint32_t)lane_base << 16) + (uint32_t)c0, v);
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = 0.f;
      }
      const int64_t nrem = p.N - (n0 + c0);
      const int nv = nrem >= 16 ? 16 : (nrem > 0 ? (int)nrem : 0);
      if (row_ok && nv > 0) p.epilogue_row(z, split, m, n0 + c0, v, nv, sq);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
  }
  if (Prob::kCtaReduce) {
    __shared__ double red[kThreads / 32];
    const double t = block_sum<kThreads>(sq, red);
    if (tid == 0) p.epilogue_cta(z, split, (int)(blockIdx.y * gridDim.x + blockIdx.x), t);
  }
}

// CTAs a launch should fill: kMinBlocks per SM
inline int ctas_target() { return kMinBlocks * kNumSMs; }

// Rows per CTA tile: the UMMA tile is always BM = 128 rows, but an M that is not a multiple of
// 128 is split into equal tiles (M = 288: 3 x 96 instead of 128 + 128 + 32), so the gathers —
// the CTA's critical path — are balanced across the launch.
inline int tile_rows(int64_t M) {
  if (M <= 0) return BM;
  const int64_t t = (M + BM - 1) / BM;
  return (int)((M + t - 1) / t);
}

template <int BN, class Prob>
void launch_tc(dpg_ctx* ctx, const Prob& p_in, int64_t batches) {
  Prob p = p_in;
  p.mstep = tile_rows(p.M);
  const int mt = (int)((p.M + p.mstep - 1) / p.mstep), nt = (int)((p.N + BN - 1) / BN);
  const int smem = Smem<BN>::FIXED + 1024 + p.scratch;
  ensure_smem_attr(reinterpret_cast<const void*>(tc_gemm_kernel<BN, Prob>), smem);
  dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)(batches * p.ksplit));
  ::dpg::launch_pdl(tc_gemm_kernel<BN, Prob>, grid, kThreads, smem, ctx->stream, p);
  DPG_LAUNCH_CHECK(ctx);
}

inline int pick_bn(int64_t n) { return n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : 128; }

// the narrowest legal UMMA N covering n (cta_group::1, M = 128: N % 16 == 0)
template <class Prob>
void launch_tc_auto(dpg_ctx* ctx, const Prob& p, int64_t batches) {
  switch (pick_bn(p.N)) {
    case 16: launch_tc<16>(ctx, p, batches); break;
    case 32: launch_tc<32>(ctx, p, batches); break;
    case 64: launch_tc<64>(ctx, p, batches); break;
    default: launch_tc<128>(ctx, p, batches); break;
  }
}

// split-K factor: only when the output tiles alone leave SMs idle; then enough splits to fill
// ksplit_ctas() CTAs with >= 2 K stages per split.
// CTAs a split-K forward / dgrad launch aims for. Two per SM: measured on the CIFAR step (fewer
// splits = less partial traffic for the reduce), 444 -> 296 CTAs took the step from 399 to
// 389 us (148: 390 us). DPG_KSPLIT=off disables split-K (the parity suite runs both ways).
inline int ksplit_ctas() {
  static const int v = [] {
    const char* e = std::getenv("DPG_KSPLIT");
    return (e && std::strcmp(e, "off") == 0) ? 0 : 2 * kNumSMs;
  }();
  return v;
}
inline int pick_ksplit(int64_t M, int64_t N, int64_t K, int64_t batches) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + 127) / 128) * batches;
  if (tiles >= kNumSMs || ksplit_ctas() == 0) return 1;
  const int64_t nk = (K + BK - 1) / BK;
  int64_t ks = (ksplit_ctas() + tiles - 1) / tiles;
  ks = std::min<int64_t>(ks, std::max<int64_t>(1, nk / 2));
  return (int)std::max<int64_t>(1, std::min<int64_t>(ks, 16));
}

}  // namespace tc
}  // namespace dpg
