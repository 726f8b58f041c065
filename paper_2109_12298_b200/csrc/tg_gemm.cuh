// tg_gemm.cuh — TMA-fed, warp-specialised tcgen05 GEMM, 3xTF32 fp32-faithful.
//
//   D[z][m][n] = sum_k A(z, m, k) * B(z, n, k)            (both operands K-major in shared memory)
//
// Operand tiles are moved by the Tensor Memory Accelerator (cp.async.bulk.tensor, tiled mode):
// the implicit im2col of a convolution is one box per (tap, channel block), whose traversal
// strides walk the convolution stride and whose out-of-bounds fill supplies the zero padding, so
// no thread computes an address or touches an operand element on its way from HBM/L2 to shared
// memory. The box lands in the canonical swizzled K-major UMMA layout (SWIZZLE_64B / 128B rows).
//
// Persistent: a CTA walks the output tiles blockIdx.x, + gridDim.x, ... (one CTA per SM), so the
// TMA producer streams the next tile's operands while the current tile's epilogue drains; the
// accumulator is double-buffered in TMEM. Warp roles (320 threads):
//   warp 0      TMA producer (one elected thread): waits for a free stage, arms its mbarrier with
//               the stage's transaction bytes, issues the boxes (Prob::issue)
//   warp 1      MMA issuer (one elected thread; also allocates TMEM): waits for a converted
//               stage, issues 3 tcgen05.mma.kind::tf32 per K = 8 slice (A_lo B_hi + A_hi B_lo +
//               A_hi B_hi) into the tile's TMEM accumulator — A read from TMEM, B from shared
//               memory — tcgen05.commit frees the stage and, after the tile's last stage, hands
//               the accumulator to the epilogue
//   warps 2-5   converters: every value of the landed fp32 tiles is split into hi = rna_tf32(x)
//               and lo = rna_tf32(x - hi), optionally scaled first (the clip factor s_n of a
//               clipped sum). A: thread = tile row (its TMEM lane), the row's BK values read from
//               the swizzled tile and written as two TMEM column blocks (tcgen05.st); B: split in
//               place, lo into a second buffer at the same swizzled offset
//
// Why A goes through TMEM: with 3 MMAs per K slice each re-reading both operands, a 128 x 64 x 32
// stage moved ~168 KB through shared memory (TMA write, converter read + 2 writes, 12 MMA operand
// reads) — bandwidth-bound at ~620 ns per stage (measured, tools/micro/tg_trace.cu). With A in
// TMEM only the TMA write, the converter's reads and B's hi/lo and MMA reads remain.
//   warps 6-9   epilogue: tcgen05.ld of TMEM lanes [32 (w % 4), +32) -> Prob::epilogue, then free
//               the accumulator buffer
//
// Rounded parts leave a zero-mean dropped lo*lo term of <= 2^-22 |x w| per product (tc_gemm.cuh's
// note on the truncated split: that one is biased and a long sum accumulates it).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "dpg_device.cuh"

namespace dpg {
namespace tg {

constexpr int BM = 128;          // UMMA M: TMEM lanes = tile rows

// Timeline trace of CTA 0 (tools/micro/tg_trace.cu builds with -DDPG_TG_TRACE): globaltimer
// stamps per role and iteration into g_tg_trace[event][iteration].
#ifdef DPG_TG_TRACE
__device__ unsigned long long g_tg_trace[10][256];
__device__ int g_tg_trace_on;  // set by the host for the one launch it traces
__device__ __forceinline__ void tg_trace(int ev, int i) {
  if (g_tg_trace_on == (int)blockIdx.x + 1 && i < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tg_trace[ev][i] = t;
  }
}
#else
__device__ __forceinline__ void tg_trace(int, int) {}
#endif

// ---- PTX wrappers ----
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
// bounded: a protocol slip (e.g. a transaction count that never completes) traps after ~2^30
// polls (tens of seconds) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
    if (done) return;
    if (n == (1u << 30)) __trap();
  }
}
// cluster-scope wait: the arrivals came from other CTAs of the cluster (release.cluster)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
    if (done) return;
    if (n == (1u << 30)) __trap();
  }
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// the shared::cluster address of this CTA's shared address a in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ float4 ld_cluster4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
// bulk copy of this CTA's shared [src, src + bytes) into another cluster CTA's shared memory,
// completing `bytes` transactions on that CTA's mbarrier (both addresses shared::cluster)
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma4(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_st2(const CUtensorMap* m, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
__device__ __forceinline__ void tma_st3(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(src)
               : "memory");
}
__device__ __forceinline__ void tma_st4(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// 16-byte chunk c of row r in a SWIZZLE_64B staging tile of 64-byte rows (matches TMA's layout)
__device__ __forceinline__ uint32_t sw64_off(int r, int c) { return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4)); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major swizzled layout of BK fp32 per row: BK = 32 -> 128 B rows (SWIZZLE_128B, UMMA layout 2),
// BK = 16 -> 64 B rows (SWIZZLE_64B, UMMA layout 4); 8-row atoms.
template <int BK>
struct KLay {
  static_assert(BK == 16 || BK == 32, "BK: one 64 B or 128 B swizzle row");
  static constexpr int ROW = BK * 4;
  static constexpr int ATOM = 8 * ROW;
  static constexpr uint64_t TYPE = BK == 32 ? 2 : 4;
  static constexpr CUtensorMapSwizzle TMA_SWIZZLE = BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  __device__ static uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(ATOM >> 4) << 32) |
           ((uint64_t)1 << 46) | (TYPE << 61);
  }
};

// kind::tf32: D f32, A/B tf32, A K-major, B K-major (or MN-major: bit 16), M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool b_mn = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
// MN-major tile of tf32 (32-bit MN-major operands need the 32-byte-atom swizzle:
// SWIZZLE_128B_BASE32B, UMMA layout 1; TMA's CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 128-byte rows of
// 32 N values, one row per K, 4-row atoms; lbo = byte stride between 32-wide N chunks, sbo = byte
// stride between 4-row K groups (CuTe's Layout_MN_SW128_32B_Atom)
__device__ __forceinline__ uint64_t desc_mn128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// issue only: the registers are valid after tcgen05.wait::ld (tmem_ld_wait)
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// this thread's TMEM lane, 16 consecutive columns from taddr
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// D[tmem] (+)= A[tmem] B[smem]^T (A K-major in TMEM: lane = row, one column per tf32 element)
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// round to nearest TF32 (ties away from zero, as cvt.rna.tf32.f32)
__device__ __forceinline__ uint32_t rna_tf32(uint32_t u) { return (u + 0x1000u) & 0xffffe000u; }

// split 16 bytes in place: hi = rna(s x) (overwrites the landed value), lo = rna(s x - hi)
template <bool kScale>
__device__ __forceinline__ void split16(uint8_t* hi, uint8_t* lo, float s) {
  float4 v = *reinterpret_cast<const float4*>(hi);
  if (kScale) {
    v.x *= s; v.y *= s; v.z *= s; v.w *= s;
  }
  uint4 h, l;
  h.x = rna_tf32(__float_as_uint(v.x)); l.x = rna_tf32(__float_as_uint(v.x - __uint_as_float(h.x)));
  h.y = rna_tf32(__float_as_uint(v.y)); l.y = rna_tf32(__float_as_uint(v.y - __uint_as_float(h.y)));
  h.z = rna_tf32(__float_as_uint(v.z)); l.z = rna_tf32(__float_as_uint(v.z - __uint_as_float(h.z)));
  h.w = rna_tf32(__float_as_uint(v.w)); l.w = rna_tf32(__float_as_uint(v.w - __uint_as_float(h.w)));
  *reinterpret_cast<uint4*>(hi) = h;
  *reinterpret_cast<uint4*>(lo) = l;
}

template <int BN, int BK, int ST, int STG, int EIN, int RED = 0>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = A_BYTES + 2 * B_BYTES;  // A (raw), B, B_lo
  static constexpr int STG_OFF = ST * STAGE;           // 2 epilogue staging buffers of STG bytes
  static constexpr int EIN_OFF = STG_OFF + 2 * STG;     // 2 epilogue input buffers of EIN bytes
  static constexpr int RED_OFF = EIN_OFF + 2 * EIN;    // split-K: peers' partial chunks (leader)
  static constexpr int CST_OFF = RED_OFF + RED;        // 2 x 256 per-tile epilogue constants
  static constexpr int BAR_OFF = CST_OFF + 2 * 1024;
  static constexpr int BARS = (3 * ST + 10) * 8;
  static constexpr int TOTAL = BAR_OFF + BARS + 16 + 1024;  // + alignment slack
};

// TMEM: two accumulator buffers of AW columns (AW = BN, or 2 BN with paired B below), then per
// stage A_hi and A_lo (BK columns each)
template <int AW, int BK, int NACC = 2>
constexpr int tmem_stage_cap() {
  return (512 - NACC * AW) / (2 * BK);
}
// deepest ring (<= 6 stages) that fits the 227 KB a CTA may use and the 512 TMEM columns
template <int BN, int BK, int STG = 0, int EIN = 0, int RED = 0, int AW = BN, int NACC = 2>
constexpr int stages_for() {
  constexpr int st = Smem<BN, BK, 1, STG, EIN>::STAGE;
  constexpr int fixed = 2 * STG + 2 * EIN + RED + 2048 + 4096;
  constexpr int lim = 227 * 1024 - fixed;
  constexpr int by_smem = (6 * st <= lim) ? 6 : (5 * st <= lim) ? 5 : (4 * st <= lim) ? 4 : (3 * st <= lim) ? 3 : 2;
  return by_smem < tmem_stage_cap<AW, BK, NACC>() ? by_smem : tmem_stage_cap<AW, BK, NACC>();
}
// Paired B (pre-split operands): B_hi and B_lo land as adjacent row blocks, so one MMA of N = 2 BN
// computes A_hi B_hi (columns [0, BN)) and A_hi B_lo ([BN, 2 BN)) and a second of N = BN adds
// A_lo B_hi into [0, BN): two MMAs per K = 8 slice instead of three. An M = 128 MMA costs the same
// 52 cycles for every N <= 64 (tools/micro/mma_rate.cu), so for the step's N = 32-64 tiles the
// wider one is free. The epilogue adds the two column blocks.
template <class Prob, int BN>
constexpr bool pair_b() {
  return Prob::kBPreSplit && !Prob::kBMajorMN && BN <= 64;  // 4 BN accumulator columns + A stages
}
template <class Prob, int BN>
constexpr int acc_width() {
  return pair_b<Prob, BN>() ? 2 * BN : BN;
}
constexpr uint32_t kTmemCols = 512;
// split-K over a cluster of CK CTAs: two chunk buffers of [128 rows][16] fp32 per peer
// staging buffers of a peer's outgoing chunks, read by rank 0 through distributed shared memory
constexpr int kRedChunk = BM * 16 * 4;
constexpr int red_bytes(int ck) { return ck > 1 ? 2 * kRedChunk : 0; }

// Tile space of a launch: mt fastest, then nt, then z.
struct Tiles {
  int m, n, z;
  __device__ int count() const { return m * n * z; }
  __device__ void at(int t, int& mt, int& nt, int& zz) const {
    mt = t % m;
    const int r = t / m;
    nt = r % n;
    zz = r / n;
  }
};

// Prob interface (all __device__ const members; the Prob is a __grid_constant__ kernel parameter,
// so tensor maps it holds are addressable by TMA):
//   static constexpr bool kScaleA;     converters multiply the A tile by scale(...)
//   int a_rows() const;                A rows that hold data (the converters write zeros past them)
//   static constexpr bool kBMajorMN;   B lands MN-major: per 32-wide N chunk one SWIZZLE_128B box of
//                                      [BK K rows][32 N] (chunks BK x 128 B apart); else K-major
//   static constexpr bool kBPreSplit;  issue() loads B_hi and B_lo (both TF32-rounded in global);
//                                      otherwise converters split the landed B in place
//   static constexpr bool kCtaReduce;  per-tile reduction of the epilogue's acc -> finish()
//   static constexpr int kStaging;     bytes of one epilogue staging buffer (per 16 columns; 0 =
//                                      the epilogue stores directly)
//   static constexpr int kEpiIn;       bytes of one epilogue input chunk loaded by TMA (0 = none)
//   int  nkb(int z) const;             K blocks of a tile of launch slice z (may be 0)
//   uint32_t stage_bytes() const;      TMA transaction bytes per stage
//   void issue(int kb, uint32_t sa, uint32_t sb, uint32_t sblo, uint32_t bar, int mt, int nt, int z) const;
//   float scale(int kb, int mt, int nt, int z) const;
//   bool has_epi_in() const;           this launch loads epilogue inputs (kEpiIn > 0)
//   uint32_t epi_in_bytes() const;     bytes one epi_load moves (<= kEpiIn)
//   void epi_load(int mt, int nt, int z, int c0, uint32_t dst, uint32_t bar) const;   kEpiIn bytes
//   uint64_t pre_epilogue(int mt, int nt, int z, int row) const;   per-thread tile state, fetched
//                                      before the accumulator is ready (e.g. a ReLU mask as bits)
//   static constexpr bool kEpiConst;   epi_const(mt, nt, z, row, float* cst) fills <= 256 per-tile
//                                      constants in shared memory (e.g. the bias of the tile's
//                                      columns) before the accumulator is ready; epilogue reads cst
//   void epilogue(int mt, int nt, int z, int row, int c0, const float (&v)[16], double& acc,
//                 uint8_t* stage, const uint8_t* in, uint64_t pre, const float* cst) const;
//                                      row < 128, columns c0 .. c0+15
//   void epi_store(int mt, int nt, int z, int c0, uint32_t stage) const;   one thread (kStaging)
//   void finish(int mt, int nt, int z, double acc_sum) const;               (kCtaReduce)
// Optional Prob members (default 0 when absent):
//   static constexpr int kTileStg;     bytes of a per-CTA tile staging area: passed to epilogue() as
//                                      `stage`, then tile_done(mt, nt, z, tid, nthreads, stage) runs
//                                      on all epilogue threads (tid < nthreads = 32 kEpiWarps)
//                                      epilogue threads after the tile's last chunk (between two
//                                      epilogue barriers), e.g. to store a re-ordered tile coalesced
//   static constexpr int kTileBlock;   > 0: blocked persistent schedule — CTA i walks a contiguous
//                                      range of tiles whose bounds are multiples of kTileBlock, so a
//                                      group of kTileBlock consecutive tiles stays on one CTA
template <class P, class = void>
struct TileStg : std::integral_constant<int, 0> {};
template <class P>
struct TileStg<P, std::void_t<decltype(P::kTileStg)>> : std::integral_constant<int, P::kTileStg> {};
template <class P, class = void>
struct TileBlock : std::integral_constant<int, 0> {};
template <class P>
struct TileBlock<P, std::void_t<decltype(P::kTileBlock)>> : std::integral_constant<int, P::kTileBlock> {};
//   static constexpr bool kAMajorMN;   A lands M-major: one unswizzled [BK K rows][BM] box (row pitch
//                                      BM x 4 bytes); the converter thread of tile row r reads column r
//                                      (a warp reads one 128-byte run per K row: conflict-free) and
//                                      applies ReLU first when a_relu() (e.g. the T > 1 linear rule's
//                                      [n][t][i] activations, i contiguous)
//   static constexpr bool kCoopStore;  with kStaging: warp-local stores instead of the leader's TMA
//                                      store — each epilogue warp stages its 32 rows of the chunk,
//                                      syncs itself (no CTA barrier, so warps do not wait on each
//                                      other) and runs coop_store(mt, nt, z, c0, row, stage) over
//                                      its own rows (e.g. STG.128 of 128-byte row segments)
template <class P, class = void>
struct CoopStore : std::false_type {};
template <class P>
struct CoopStore<P, std::void_t<decltype(P::kCoopStore)>> : std::integral_constant<bool, P::kCoopStore> {};
//   static constexpr int kAccBufs;     TMEM accumulator buffers, 2 (default: a tile's epilogue overlaps
//                                      the next tile's MMAs) or 1 (a 256-column tile; the next tile's
//                                      MMAs wait for the epilogue's TMEM reads)
template <class P, class = void>
struct AccBufs : std::integral_constant<int, 2> {};
template <class P>
struct AccBufs<P, std::void_t<decltype(P::kAccBufs)>> : std::integral_constant<int, P::kAccBufs> {};
//   static constexpr bool kBRawMN;     (with kAMajorMN, kBMajorMN = false, 8 converter warps, BK = 32,
//                                      BN = 128) B lands as ONE unswizzled [BK][BN] box (N
//                                      contiguous) in the B_lo buffer; converter warps 6-9 transpose
//                                      it into K-major SWIZZLE_128B rows of B_hi / B_lo (thread = B
//                                      row), warps 2-5 convert A. One 512-byte-row box instead of
//                                      BN / 32 swizzled 128-byte-row boxes: fewer TMA requests
template <class P, class = void>
struct BRawMN : std::false_type {};
template <class P>
struct BRawMN<P, std::void_t<decltype(P::kBRawMN)>> : std::integral_constant<bool, P::kBRawMN> {};
template <class P, class = void>
struct AMajorMN : std::false_type {};
template <class P>
struct AMajorMN<P, std::void_t<decltype(P::kAMajorMN)>> : std::integral_constant<bool, P::kAMajorMN> {};

//   static constexpr int kConvWarps;   converter warps, 4 (default) or 8 (two per TMEM lane quarter,
//                                      splitting the A columns; for operands both split on the fly)
template <class P, class = void>
struct ConvWarps : std::integral_constant<int, 4> {};
template <class P>
struct ConvWarps<P, std::void_t<decltype(P::kConvWarps)>> : std::integral_constant<int, P::kConvWarps> {};
//   static constexpr int kEpiWarps;    epilogue warps, 4 (default) or 8: two per TMEM lane quarter,
//                                      taking alternate 16-column chunks (for latency-bound
//                                      epilogues; plain or warp-local-store epilogues only)
template <class P, class = void>
struct EpiWarps : std::integral_constant<int, 4> {};
template <class P>
struct EpiWarps<P, std::void_t<decltype(P::kEpiWarps)>> : std::integral_constant<int, P::kEpiWarps> {};
// epilogue warps of a launch: a cluster split-K launch keeps 4 (its exchange is per lane quarter)
template <class P, int CK>
constexpr int epi_warps() {
  return CK > 1 ? 4 : EpiWarps<P>::value;
}
// producer + MMA warps, the converters, the epilogue warps
template <class P, int CK = 1>
constexpr int threads_of() {
  return 64 + 32 * ConvWarps<P>::value + 32 * epi_warps<P, CK>();
}
// Smem's STG: half the epilogue staging bytes (it reserves two). Warp-local stores need one chunk
// slot per epilogue warp group (each warp touches only its own rows, and rewrites them only
// after its own reads); the leader's TMA stores double-buffer one slot.
template <class P>
constexpr int stg_bytes() {
  return CoopStore<P>::value ? P::kStaging * (EpiWarps<P>::value / 4) / 2 : P::kStaging;
}
constexpr int kEpiThreads = 128;
//
// Split-K over a thread-block cluster (CK > 1): the CK CTAs of a cluster own one tile at a time,
// CTA rank r running K blocks [r nkb / CK, (r + 1) nkb / CK) into its own TMEM accumulator. Per
// 16-column chunk the peers store their partial through distributed shared memory into the rank-0
// CTA's reduction buffer (st.shared::cluster, then a remote mbarrier arrive); rank 0 adds them in
// rank order (deterministic), frees the buffer with a remote arrive per peer, and runs the epilogue.
template <int BN, int BK, int ST, class Prob, int CK = 1>
__global__ void __launch_bounds__(threads_of<Prob, CK>(), 1) tg_kernel(const __grid_constant__ Prob p, const Tiles tiles) {
  constexpr int STG = stg_bytes<Prob>(), EIN = Prob::kEpiIn;
  constexpr int EW = epi_warps<Prob, CK>(), EH = EW / 4;  // epilogue warps, chunk interleave
  static_assert(CK == 1 || (EIN == 0 && !Prob::kCtaReduce), "cluster split-K: plain epilogues only");
  constexpr int TST = TileStg<Prob>::value, TBL = TileBlock<Prob>::value;
  constexpr int CW = ConvWarps<Prob>::value, kCvt = 32 * CW;
  constexpr bool BRAW = BRawMN<Prob>::value;
  static_assert(!BRAW || (AMajorMN<Prob>::value && !Prob::kBMajorMN && !Prob::kBPreSplit && CW >= 8 && BK == 32 &&
                          BN == 128),
                "raw MN-major B: M-major A, K-major B for the MMA, 8 or 16 converter warps, BK 32, BN 128");
  // raw B: converter warp groups [0, CG) convert A, [CG, 2 CG) transpose B (CG = CW / 8 groups of 4
  // warps each; with two groups per operand, each takes half of the 32 columns / K values)
  constexpr int CG = CW / 8;
  static_assert(CW == 4 || CW == 8 || CW == 16, "converter warps: 4, 8 or 16");
  static_assert(EW == 4 || ((EW == 8 || EW == 16) && CK == 1 && EIN == 0 &&
                            (STG == 0 || CoopStore<Prob>::value)),
                "8 epilogue warps: plain or warp-local-store epilogues only");
  static_assert(TBL == 0 || CK == 1, "blocked tile schedule: no cluster split");
  using S = Smem<BN, BK, ST, STG, EIN, red_bytes(CK) + TST>;
  using Lay = KLay<BK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = su32(smem);
  const uint32_t bar0 = sbase + S::BAR_OFF;  // full[ST], conv[ST], empty[ST], tfull[2], tempty[2], ein[2]
  auto full = [&](int s) { return bar0 + 8u * s; };
  auto conv = [&](int s) { return bar0 + 8u * (ST + s); };
  auto empty = [&](int s) { return bar0 + 8u * (2 * ST + s); };
  auto tfull = [&](int a) { return bar0 + 8u * (3 * ST + a); };
  auto tempty = [&](int a) { return bar0 + 8u * (3 * ST + 2 + a); };
  auto ein = [&](int a) { return bar0 + 8u * (3 * ST + 4 + a); };
  auto red_full = [&](int a) { return bar0 + 8u * (3 * ST + 6 + a); };   // rank 0: peers' chunks landed
  auto red_empty = [&](int a) { return bar0 + 8u * (3 * ST + 8 + a); };  // peers: rank 0 read them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::BAR_OFF + S::BARS);
  auto sA = [&](int s) { return sbase + s * S::STAGE; };
  auto sB = [&](int s) { return sbase + s * S::STAGE + S::A_BYTES; };
  auto sBlo = [&](int s) { return sbase + s * S::STAGE + S::A_BYTES + S::B_BYTES; };
  // TMEM columns of stage s's A_hi / A_lo (after the two accumulator buffers)
  constexpr bool PAIR = pair_b<Prob, BN>();
  constexpr int AW = acc_width<Prob, BN>();
  constexpr int NACC = AccBufs<Prob>::value;
  static_assert(NACC == 1 || NACC == 2, "one or two accumulator buffers");
  static_assert(ST >= 2 && NACC * AW + ST * 2 * BK <= 512, "TMEM: accumulators + A stages exceed 512 columns");
  auto tA = [&](int s) { return (uint32_t)(NACC * AW + s * 2 * BK); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = tiles.count();
  const int crank = CK > 1 ? (int)cluster_rank() : 0;
  int t_first = CK > 1 ? (int)blockIdx.x / CK : (int)blockIdx.x;
  int t_step = CK > 1 ? (int)gridDim.x / CK : (int)gridDim.x;
  int t_end = ntiles;
  if constexpr (TBL > 0) {  // contiguous, kTileBlock-aligned range of tiles per CTA
    const int groups = (ntiles + TBL - 1) / TBL;
    t_first = (int)((int64_t)groups * blockIdx.x / gridDim.x) * TBL;
    t_end = std::min(ntiles, (int)((int64_t)groups * (blockIdx.x + 1) / gridDim.x) * TBL);
    t_step = 1;
  }
  // this CTA's K blocks of a tile of slice z: [kb0, kb0 + nk)
  auto krange = [&](int z, int& kb0, int& nk) {
    const int n = p.nkb(z);
    kb0 = CK > 1 ? n * crank / CK : 0;
    nk = CK > 1 ? n * (crank + 1) / CK - kb0 : n;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full(s), 1);
      mbar_init(conv(s), kCvt);
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 32 * EW);
      mbar_init(ein(a), 1);
      mbar_init(red_full(a), (CK - 1) * kEpiThreads);  // every peer epilogue thread, per chunk
      mbar_init(red_empty(a), kEpiThreads);            // every rank-0 epilogue thread, per use
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CK > 1) cluster_sync_all();  // every CTA's barriers exist before remote arrives
  tc_fence_after();
  pdl_wait();  // barrier init and TMEM allocation overlap the previous kernel's tail
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = t_first; t < t_end; t += t_step) {
        int mt, nt, z;
        tiles.at(t, mt, nt, z);
        int kb0, nkb;
        krange(z, kb0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % ST;
          if (it >= ST) mbar_wait(empty(s), ((it / ST) - 1) & 1);
          tg_trace(0, it);
          mbar_expect_tx(full(s), p.stage_bytes());
          p.issue(kb0 + kb, sA(s), sB(s), sBlo(s), full(s), mt, nt, z);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(BN, Prob::kBMajorMN);
      constexpr uint32_t idesc2 = idesc_tf32(PAIR ? 2 * BN : BN, Prob::kBMajorMN);
      int it = 0, j = 0;
      for (int t = t_first; t < t_end; t += t_step, ++j) {
        int mt, nt, z;
        tiles.at(t, mt, nt, z);
        int kb0, nkb;
        krange(z, kb0, nkb);
        const int a = j % NACC;
        if (j >= NACC) mbar_wait(tempty(a), ((j / NACC) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(a * AW);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(conv(s), (it / ST) & 1);
          tg_trace(3, it);
          tc_fence_after();
          const uint32_t ahi = tmem + tA(s), alo = ahi + BK;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
            uint64_t bhi, blo;
            if constexpr (Prob::kBMajorMN) {  // B as [BK rows][BN] in 32-wide N chunks of BK rows
              bhi = desc_mn128(sB(s) + kk * 1024, BK * 128, 512);
              blo = desc_mn128(sBlo(s) + kk * 1024, BK * 128, 512);
            } else {
              const uint32_t off = kk * 32;  // 8 tf32 = 32 B along the swizzled row
              bhi = Lay::desc(sB(s) + off);
              blo = Lay::desc(sBlo(s) + off);
            }
            if constexpr (PAIR) {  // [A_hi B_hi | A_hi B_lo], then A_lo B_hi into the first block
              mma_tf32_ts(acc, ahi + kk * 8, bhi, idesc2, acc0);
              mma_tf32_ts(acc, alo + kk * 8, bhi, idesc, 1u);
            } else {
              mma_tf32_ts(acc, alo + kk * 8, bhi, idesc, acc0);
              mma_tf32_ts(acc, ahi + kk * 8, blo, idesc, 1u);
              mma_tf32_ts(acc, ahi + kk * 8, bhi, idesc, 1u);
            }
          }
          mma_commit(empty(s));
        }
        mma_commit(tfull(a));
      }
    }
  } else if (warp < 2 + CW) {
    // converters. A: thread = row 32 (w % 4) + lane of the tile (its TMEM lane)
    const int tc = threadIdx.x - 64;
    const int q = warp & 3;
    const int h0 = (warp - 2) >> 2;  // 8 converter warps: two per lane quarter, alternate 16-column halves
    const int r = 32 * q + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * q) << 16);
    int it = 0;
    for (int t = t_first; t < t_end; t += t_step) {
      int mt, nt, z;
      tiles.at(t, mt, nt, z);
      int kb0, nkb;
      krange(z, kb0, nkb);
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % ST;
        mbar_wait(full(s), (it / ST) & 1);
        if (tc == 0) tg_trace(1, it);
        float sc = 1.f;
        if (Prob::kScaleA) sc = p.scale(kb0 + kb, mt, nt, z);
        if constexpr (BRAW) {
          if (h0 >= CG) {
            // B: row r of the tile is column r of the landed [BK][BN] box; read this group's K
            // range of it (every B thread reads before any writes: the raw box sits in the B_lo
            // buffer), then split and write K-major SWIZZLE_128B row chunks (16 B, chunk c at
            // c ^ (r & 7))
            constexpr int KB = BK / CG;  // K values per B group
            const int k0 = (h0 - CG) * KB;
            uint8_t* bhi = smem + s * S::STAGE + S::A_BYTES;
            uint8_t* blo = bhi + S::B_BYTES;
            const float* bcol = reinterpret_cast<const float*>(blo) + r;
            float e[KB];
#pragma unroll
            for (int u = 0; u < KB; ++u) e[u] = bcol[(k0 + u) * BN];
            asm volatile("bar.sync 2, %0;" ::"n"(128 * CG) : "memory");  // every B warp has read the box
#pragma unroll
            for (int cc = 0; cc < KB / 4; ++cc) {
              const int c = k0 / 4 + cc;
              uint4 hv, lv;
              uint32_t* hp = reinterpret_cast<uint32_t*>(&hv);
              uint32_t* lp = reinterpret_cast<uint32_t*>(&lv);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                hp[u] = rna_tf32(__float_as_uint(e[4 * cc + u]));
                lp[u] = rna_tf32(__float_as_uint(e[4 * cc + u] - __uint_as_float(hp[u])));
              }
              const uint32_t off = (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4));
              *reinterpret_cast<uint4*>(bhi + off) = hv;
              *reinterpret_cast<uint4*>(blo + off) = lv;
            }
          }
        }
        if constexpr (AMajorMN<Prob>::value) {  // [BK][BM] box: this thread's column r
          const float* acol = reinterpret_cast<const float*>(smem + s * S::STAGE) + r;
          const bool relu = p.a_relu();
#pragma unroll
          for (int h = BRAW ? h0 : h0; h < (BRAW && h0 >= CG ? 0 : BK / 16); h += BRAW ? CG : CW / 4) {
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              float e = acol[(16 * h + u) * BM];
              if (relu) e = e > 0.f ? e : 0.f;
              if (Prob::kScaleA) e *= sc;
              hi[u] = rna_tf32(__float_as_uint(e));
              lo[u] = rna_tf32(__float_as_uint(e - __uint_as_float(hi[u])));
            }
            tmem_st16(lane_addr + tA(s) + 16 * h, hi);
            tmem_st16(lane_addr + tA(s) + BK + 16 * h, lo);
          }
        }
        const uint8_t* arow = smem + s * S::STAGE + r * Lay::ROW;
        const int sw = Lay::ROW == 128 ? (r & 7) : ((r >> 1) & 3);
#pragma unroll
        for (int h = h0; h < (AMajorMN<Prob>::value ? 0 : BK / 16); h += CW / 4) {  // 16 columns (4 chunks) at a time
          uint32_t hi[16], lo[16];
          const bool zero_row = r >= p.a_rows();  // rows past the operand: zeros (no stale data)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float4 v = *reinterpret_cast<const float4*>(arow + (((4 * h + c) ^ sw) << 4));
            if (zero_row) v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (Prob::kScaleA) {
              v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
            }
            const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              hi[4 * c + u] = rna_tf32(__float_as_uint(e[u]));
              lo[4 * c + u] = rna_tf32(__float_as_uint(e[u] - __uint_as_float(hi[4 * c + u])));
            }
          }
          tmem_st16(lane_addr + tA(s) + 16 * h, hi);
          tmem_st16(lane_addr + tA(s) + BK + 16 * h, lo);
        }
        if (BRAW) {
          fence_proxy_async();  // the transposed B rows, for the MMA's async-proxy reads
        } else if (!Prob::kBPreSplit) {
          uint8_t* b = smem + s * S::STAGE + S::A_BYTES;
#pragma unroll 4
          for (int i = tc * 16; i < S::B_BYTES; i += kCvt * 16) split16<false>(b + i, b + S::B_BYTES + i, 1.f);
          fence_proxy_async();
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        if (tc == 0) tg_trace(2, it);
        mbar_arrive(conv(s));
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes [32 (w % 4), +32) of the tile's accumulator buffer;
    // outputs staged in shared memory go out as TMA bulk stores issued by one thread
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const bool leader = warp == 2 + CW && lane == 0;
    const int ew = warp - (2 + CW), eh = ew >> 2;  // epilogue warp, its chunk phase
    int j = 0, g = 0;  // tile and chunk counters of this CTA
    for (int t = t_first; t < t_end; t += t_step, ++j) {
      int mt, nt, z;
      tiles.at(t, mt, nt, z);
      int kb0, nkb;
      krange(z, kb0, nkb);
      const int a = j % NACC;
      const bool epi_in = EIN > 0 && p.has_epi_in();
      if (epi_in && leader) {  // epilogue inputs of the tile's first chunk
        mbar_expect_tx(ein(g & 1), p.epi_in_bytes());
        p.epi_load(mt, nt, z, 0, sbase + S::EIN_OFF + (g & 1) * EIN, ein(g & 1));
      }
      const uint64_t pre = crank == 0 ? p.pre_epilogue(mt, nt, z, row) : 0;  // overlaps the tile's MMAs
      float* cst = reinterpret_cast<float*>(smem + S::CST_OFF + a * 1024);
      if constexpr (Prob::kEpiConst) {
        if (crank == 0) p.epi_const(mt, nt, z, row, cst);
      }
      mbar_wait(tfull(a), (j / NACC) & 1);
      if constexpr (Prob::kEpiConst) asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // constants written
      if (row == 0) tg_trace(4, j);
      tc_fence_after();
      if (t + t_step >= t_end) pdl_trigger();  // last tile: the next kernel may launch
      double acc = 0.0;
      float v[16];
      uint32_t vn[16];  // the next chunk, in flight from TMEM while this one is processed
      uint32_t vm[16];  // paired B: the A_hi B_lo block of the same columns
      const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * AW);
#pragma unroll 1
      for (int c0 = 16 * eh; c0 < BN; c0 += 16 * EH, ++g) {
        if (epi_in && leader && c0 + 16 < BN) {  // prefetch the next chunk's inputs
          mbar_expect_tx(ein((g + 1) & 1), p.epi_in_bytes());
          p.epi_load(mt, nt, z, c0 + 16, sbase + S::EIN_OFF + ((g + 1) & 1) * EIN, ein((g + 1) & 1));
        }
        if (nkb > 0) {
          if (c0 == 16 * eh) {
            tmem_ld16_async(trow + (uint32_t)c0, vn);
            if constexpr (PAIR) tmem_ld16_async(trow + (uint32_t)(BN + c0), vm);
          }
          tmem_ld_wait();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            v[jj] = PAIR ? __uint_as_float(vn[jj]) + __uint_as_float(vm[jj]) : __uint_as_float(vn[jj]);
          if (c0 + 16 * EH < BN) {
            tmem_ld16_async(trow + (uint32_t)(c0 + 16 * EH), vn);
            if constexpr (PAIR) tmem_ld16_async(trow + (uint32_t)(BN + c0 + 16 * EH), vm);
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) v[jj] = 0.f;
        }
        if (row == 0) tg_trace(6, j * 8 + c0 / 16);
        if (c0 + 16 * EH >= BN) {  // every TMEM read of this buffer is done (waited): release it
          tc_fence_before();
          mbar_arrive(tempty(a));
        }
        if constexpr (CK > 1) {  // split-K partials: rank 0 pulls the peers' chunks, adds in rank order
          const int bb = g & 1;
          const uint32_t send = sbase + S::RED_OFF + bb * kRedChunk + row * 64;  // [2][128][16]
          if (crank != 0) {
            // peer: stage the chunk in local shared memory, then tell rank 0 it is there
            if (g >= 2) mbar_wait_cluster(red_empty(bb), ((g >> 1) - 1) & 1);  // rank 0 read it
            float4* st4 = reinterpret_cast<float4*>(smem + (send - sbase));
#pragma unroll
            for (int c = 0; c < 4; ++c) st4[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            mbar_arrive_remote(mapa(red_full(bb), 0));  // per thread: releases its own row
            if (row == 0) tg_trace(8, j * 8 + c0 / 16);
            continue;  // the epilogue is rank 0's
          }
          mbar_wait_cluster(red_full(bb), (g >> 1) & 1);
          if (row == 0) tg_trace(8, j * 8 + c0 / 16);
          float4 w[CK - 1][4];
#pragma unroll
          for (int r = 1; r < CK; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) w[r - 1][c] = ld_cluster4(mapa(send + 16 * c, (uint32_t)r));
#pragma unroll
          for (int r = 1; r < CK; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              v[4 * c] += w[r - 1][c].x; v[4 * c + 1] += w[r - 1][c].y;
              v[4 * c + 2] += w[r - 1][c].z; v[4 * c + 3] += w[r - 1][c].w;
            }
#pragma unroll
          for (int r = 1; r < CK; ++r) mbar_arrive_remote(mapa(red_empty(bb), (uint32_t)r));  // row read
        }
        const uint8_t* in = nullptr;
        if (epi_in) {
          mbar_wait(ein(g & 1), (g >> 1) & 1);
          in = smem + S::EIN_OFF + (g & 1) * EIN;
        }
        uint8_t* stg = STG > 0   ? smem + S::STG_OFF + (CoopStore<Prob>::value ? eh * Prob::kStaging : (g & 1) * STG)
                       : TST > 0 ? smem + S::RED_OFF + red_bytes(CK)
                                 : nullptr;
        p.epilogue(mt, nt, z, row, c0, v, acc, stg, in, pre, cst);
        if constexpr (STG > 0 && CoopStore<Prob>::value) {
          // this warp's rows are staged; the warp alone reads them back and stores them (the
          // buffer is rewritten by the same warp two chunks later, after these reads)
          __syncwarp();
          p.coop_store(mt, nt, z, c0, row, stg);
          __syncwarp();
        } else if (STG > 0) {
          fence_proxy_async();
          if (leader) bulk_wait_read<0>();  // the previous chunk's stores have read their buffer
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (leader) {
            p.epi_store(mt, nt, z, c0, sbase + S::STG_OFF + (g & 1) * STG);
            bulk_commit();
          }
        } else if (epi_in) {
          asm volatile("bar.sync 1, 128;" ::: "memory");  // the input buffer may be refilled
        }
        if (row == 0) tg_trace(7, j * 8 + c0 / 16);
      }
      if (row == 0) tg_trace(5, j);
      if (Prob::kCtaReduce) {
        __shared__ double red[2][16];
        acc = warp_sum(acc);
        const int rb = j & 1;  // alternate per tile (also with one accumulator buffer)
        if (lane == 0) red[rb][eh * 4 + q] = acc;  // summed in lane-quarter order below
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
        if (ew == 0 && lane == 0) {
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < EW; ++w) sum += red[rb][w];
          p.finish(mt, nt, z, sum);
        }
      }
      if constexpr (TST > 0) {
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // every chunk of the tile is staged
        p.tile_done(mt, nt, z, 32 * ew + lane, 32 * EW, smem + S::RED_OFF + red_bytes(CK));
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");  // staging free for the next tile
      }
    }
    if (((STG > 0 && !CoopStore<Prob>::value) || CK > 1) && leader) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CK > 1) cluster_sync_all();  // no CTA leaves while a peer may still address it
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---- host side: tensor maps ----
// Tiled fp32 tensor map. dims / strides innermost first (strides in bytes, for dims 1..rank-1);
// box and traversal strides (estr: 1, or the convolution stride) per dim.
CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box, const uint32_t* estr, CUtensorMapSwizzle swz);

#ifdef DPG_TG_TRACE
inline int& trace_launch_count() {
  static int n = 0;
  return n;
}
#endif

// clusters of `ck` CTAs of fn (smem bytes each) that fit the GPU at once (cached per device)
int max_active_clusters(const void* fn, int smem, int ck, int threads);

// grid: the tile space (m tiles, n tiles, slices); the launch is persistent, min(tiles, #SMs) CTAs
// (CK > 1: min(tiles, co-resident clusters) clusters of CK CTAs)
template <int BN, int BK, int ST, class Prob, int CK = 1>
void launch(dpg_ctx* ctx, const Prob& p, dim3 grid) {
  const int smem = Smem<BN, BK, ST, stg_bytes<Prob>(), Prob::kEpiIn, red_bytes(CK) + TileStg<Prob>::value>::TOTAL;
  const void* fn = reinterpret_cast<const void*>(tg_kernel<BN, BK, ST, Prob, CK>);
  ensure_smem_attr(fn, smem);
  const Tiles tiles{(int)grid.x, (int)grid.y, (int)grid.z};
  const int64_t nt = (int64_t)grid.x * grid.y * grid.z;
  const int64_t slots = CK > 1 ? max_active_clusters(fn, smem, CK, threads_of<Prob, CK>()) : kNumSMs;
  const unsigned ctas = (unsigned)(std::min<int64_t>(nt, std::max<int64_t>(slots, 1)) * CK);
  if (std::getenv("DPG_TG_VERBOSE"))
    std::fprintf(stderr, "tg launch BN=%d BK=%d ST=%d CK=%d tiles=%lld slots=%lld ctas=%u smem=%d\n", BN, BK, ST, CK,
                 (long long)nt, (long long)slots, ctas, smem);
#ifdef DPG_TG_TRACE
  {  // trace only the DPG_TG_TRACE_AT-th TMA-fed launch of the process
    const int at = std::getenv("DPG_TG_TRACE_AT") ? std::atoi(std::getenv("DPG_TG_TRACE_AT")) : -1;
    const char* cta = std::getenv("DPG_TG_TRACE_CTA");  // the traced CTA (default 0)
    const int on = trace_launch_count()++ == at ? 1 + (cta ? std::atoi(cta) : 0) : 0;
    cudaMemcpyToSymbolAsync(g_tg_trace_on, &on, sizeof(int), 0, cudaMemcpyHostToDevice, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
  }
#endif
  if constexpr (CK == 1) {
    ::dpg::launch_pdl(tg_kernel<BN, BK, ST, Prob>, dim3(ctas), threads_of<Prob, CK>(), smem, ctx->stream, p, tiles);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(threads_of<Prob, CK>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CK;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    (void)cudaLaunchKernelEx(&cfg, tg_kernel<BN, BK, ST, Prob, CK>, p, tiles);
  }
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace tg
}  // namespace dpg
