// tg_linear.cu — the T > 1 linear contractions on the TMA-fed tcgen05 core (tg_gemm.cuh), the
// "genuinely dense" per-sample path of BASELINE configs[1] (Linear 512 -> 512, T = 64, b = 256).
//
//   rule        G[n][o][i] = sum_t relu?(A[n][t][i]) H[n][t][o]           grad_sample.hpp:53-59,
//                                                                         tensor.hpp:303-338
//   clipped sum S[o][i]    = sum_(n, t) s_n relu?(A[n][t][i]) H[n][t][o]  optimizer.hpp:100-114
//                            as (s . H)^T A, split over samples, partials summed in split order
//
// Tile rows (TMEM lanes) are the input index i, columns the output index o, so an epilogue warp's
// store of one column is 32 consecutive i of the reference-layout [o][i] gradient: one full
// 128-byte line per store instruction. Both operands are plain row-major activations: A lands
// M-major as one [BK t][128 i] box (the converters read a column per thread, apply ReLU and the
// clip factor, split into TF32 hi / lo in TMEM), H lands MN-major as [BK t][32 o] boxes with the
// 32-byte-atom swizzle and is split in place. Tensor maps are 3-D ([n][t][feature]), so a K block
// never crosses a sample: rows past T come from the out-of-bounds zero fill, and any T works.
#include <algorithm>
#include <cstdlib>

#include "tg_gemm.cuh"

namespace dpg {
namespace tg {

#ifndef DPG_TG_LIN_BRAW
#define DPG_TG_LIN_BRAW 1
#endif
#ifndef DPG_TG_LIN_CSUM_CW
#define DPG_TG_LIN_CSUM_CW 8
#endif
#ifndef DPG_TG_LIN_EW
#define DPG_TG_LIN_EW 16
#endif

namespace {
constexpr int kLinBN = 128;  // clipped sum tile width; the rule takes 256 where r allows (below)

// one K block = BK time steps of one sample; tiles of 128 i x BN o
template <int BK, int BN>
struct LinBase {
  static constexpr bool kBPreSplit = false, kBMajorMN = true, kAMajorMN = true, kEpiConst = false;
  // both operands split on the fly: two converter warps per TMEM lane quarter (the clipped sum's
  // stage rate depends on them; the rule trades them for epilogue warps, below)
  static constexpr int kConvWarps = 8;
  // a 16-column chunk of the tile is transposed through shared memory ([16 o][128 i]) and leaves
  // as 512-byte runs: one STG.128 per thread and column (measured: one 4-byte column store per
  // thread, or a TMA bulk store of the staged chunk, drain at 1-2 TB/s)
  static constexpr int kStaging = 16 * BM * 4, kEpiIn = 0;
  static constexpr bool kCoopStore = true;
  CUtensorMap ma, mb;  // A: {d, T, b} box {128, BK, 1}; H: {r, T, b} box {32, BK, 1}
  float* out;          // [slices][r][d]; null: norms only (no per-sample gradient)
  bool stream;         // streaming stores (the per-sample record) or L2-resident (partials)
  int d, r, T, b, relu;
  __device__ bool a_relu() const { return relu != 0; }
  __device__ int a_rows() const { return BM; }
  __device__ uint32_t stage_bytes() const { return (uint32_t)((BM + BN) * BK * 4); }
  __device__ void load(int n, int tb, uint32_t sa, uint32_t sb, uint32_t bar, int mt, int nt) const {
    tma3(sa, &ma, bar, mt * BM, tb * BK, n);
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) tma3(sb + c * (BK * 128), &mb, bar, nt * BN + 32 * c, tb * BK, n);
  }
  __device__ bool has_epi_in() const { return false; }
  __device__ uint32_t epi_in_bytes() const { return 0; }
  __device__ void epi_load(int, int, int, int, uint32_t, uint32_t) const {}
  __device__ uint64_t pre_epilogue(int, int, int, int) const { return 0; }
  __device__ void epi_const(int, int, int, int, float*) const {}
  // the chunk's 16 columns, transposed through shared memory: stage[j][row] (consecutive rows,
  // conflict-free)
  __device__ static void stage16(uint8_t* stage, int row, const float (&v)[16]) {
    float* st = reinterpret_cast<float*>(stage);
#pragma unroll
    for (int j = 0; j < 16; ++j) st[j * BM + row] = v[j];
  }
  __device__ void epi_store(int, int, int, int, uint32_t) const {}
  // this warp's [16 o][32 i] block (rows 32 q .. 32 q + 31 of every staged o row): lane l stores
  // o = l / 8 + 4 k, i = 32 q + 4 (l % 8): one STG.128 covers four 128-byte row segments
  __device__ void coop_store(int mt, int nt, int z, int c0, int row, const uint8_t* stage) const {
    if (!out) return;
    const float4* st = reinterpret_cast<const float4*>(stage);
    const int q = row >> 5, l = row & 31;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ol = (l >> 3) + 4 * k, il = 32 * q + 4 * (l & 7);
      const int i = mt * BM + il, o = nt * BN + c0 + ol;
      const float4 v = st[(ol * BM + il) >> 2];
      if (o < r && i < d) {
        float* p = out + ((int64_t)z * r + o) * d + i;
        if (stream) st_stream4(p, v);
        else *reinterpret_cast<float4*>(p) = v;
      }
    }
  }
};

// per-sample rule: slice z = sample n; fused squared norm per (tile, sample). BN = 256: one
// accumulator buffer of 256 columns (the 128 columns of a second would leave no room for the A
// stages), so the tile's epilogue and the next tile's MMAs alternate — the epilogue's TMEM reads
// then run without concurrent MMAs, and A is loaded and converted once per 256 outputs
template <int BK, int BN>
struct LinRuleT : LinBase<BK, BN> {
  static constexpr bool kScaleA = false, kCtaReduce = true;
  static constexpr int kAccBufs = BN > 128 ? 1 : 2;
  // the epilogue's per-chunk chain (TMEM load, staging, 16-byte stores) is latency-bound: four
  // warps per lane quarter take interleaved chunks (DPG_TG_LIN_EW=4|8 at build time: one | two);
  // 16 epilogue warps leave registers for 4 converter warps (704 threads)
  static constexpr int kEpiWarps = DPG_TG_LIN_EW;
  static constexpr int kConvWarps = DPG_TG_LIN_EW > 8 ? 4 : 8;
  double* sq;
  int mtiles, nrows128;  // norm slab rows are per 128-wide n tile (tc::gs_linear_rows)
  __device__ int nkb(int) const { return (this->T + BK - 1) / BK; }
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t, uint32_t bar, int mt, int nt, int z) const {
    this->load(z, kb, sa, sb, bar, mt, nt);
  }
  __device__ float scale(int, int, int, int) const { return 1.f; }
  // rows / columns past d / r hold exact zeros (zero-filled operands), so the norm needs no mask
  __device__ void epilogue(int, int, int, int row, int, const float (&v)[16], double& acc, uint8_t* stage,
                           const uint8_t*, uint64_t, const float*) const {
    if (this->out) this->stage16(stage, row, v);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      a0 += (double)v[j] * v[j];
      a1 += (double)v[j + 1] * v[j + 1];
      a2 += (double)v[j + 2] * v[j + 2];
      a3 += (double)v[j + 3] * v[j + 3];
    }
    acc += (a0 + a1) + (a2 + a3);
  }
  // norm row = 128-wide n tile * m tiles + m tile (tc::gs_linear_rows' order); a 256-wide tile
  // puts its sum in its first row and zero in its second
  __device__ void finish(int mt, int nt, int z, double s) const {
    if (!sq) return;
    constexpr int R = BN / 128;
#pragma unroll
    for (int h = 0; h < R; ++h)
      if (nt * R + h < nrows128) sq[(int64_t)((nt * R + h) * mtiles + mt) * this->b + z] = h == 0 ? s : 0.0;
  }
};

// clipped sum: slice z = samples [z spl, z spl + spl); partial [z][o][i]
// (kBRawMN: H lands as one unswizzled [BK][128] box in the B_lo buffer and the converters
// transpose it into K-major B_hi / B_lo rows — 1 TMA box per stage instead of 4 swizzled ones; the
// clipped sum's stage rate is TMA-bound, ~4 ns per 128-byte request per SM)
template <int BK>
struct LinCsumT : LinBase<BK, kLinBN> {
  static constexpr bool kScaleA = true, kCtaReduce = false;
  static constexpr bool kBRawMN = DPG_TG_LIN_BRAW != 0 && BK == 32, kBMajorMN = !kBRawMN;
  CUtensorMap mh;  // kBRawMN: H as {r, T, b} box {128, BK, 1}, unswizzled
  // converter warps (DPG_TG_LIN_CSUM_CW=16 at build time: two groups per operand, measured
  // 90 -> 94 us: the stage rate is not conversion-bound)
  static constexpr int kConvWarps = kBRawMN ? DPG_TG_LIN_CSUM_CW : 8;
  const float* svec;
  int spl, kpt;
  __device__ int nkb(int z) const {
    const int ns = min(spl, this->b - z * spl);
    return ns > 0 ? ns * kpt : 0;
  }
  __device__ void issue(int kb, uint32_t sa, uint32_t sb, uint32_t sblo, uint32_t bar, int mt, int nt, int z) const {
    const int n = z * spl + kb / kpt, tb = kb % kpt;
    if constexpr (kBRawMN) {
      tma3(sa, &this->ma, bar, mt * BM, tb * BK, n);
      tma3(sblo, &mh, bar, nt * kLinBN, tb * BK, n);
    } else {
      this->load(n, tb, sa, sb, bar, mt, nt);
    }
  }
  __device__ float scale(int kb, int, int, int z) const { return __ldg(svec + z * spl + kb / kpt); }
  __device__ void epilogue(int, int, int, int row, int, const float (&v)[16], double&, uint8_t* stage,
                           const uint8_t*, uint64_t, const float*) const {
    this->stage16(stage, row, v);
  }
  __device__ void finish(int, int, int, double) const {}
};

int pick_bk(int64_t mid) { return mid <= 16 ? 16 : 32; }

template <int BK, class Pr>
void set_maps(Pr& p, const float* acts, const float* hw, int64_t b, int64_t mid, int64_t d, int64_t r) {
  const uint64_t da[3] = {(uint64_t)d, (uint64_t)mid, (uint64_t)b};
  const uint64_t sa[2] = {(uint64_t)d * 4, (uint64_t)(mid * d * 4)};
  const uint32_t ba[3] = {(uint32_t)BM, (uint32_t)BK, 1};
  p.ma = make_map(acts, 3, da, sa, ba, nullptr, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t dh[3] = {(uint64_t)r, (uint64_t)mid, (uint64_t)b};
  const uint64_t sh[2] = {(uint64_t)r * 4, (uint64_t)(mid * r * 4)};
  const uint32_t bh[3] = {32, (uint32_t)BK, 1};
  p.mb = make_map(hw, 3, dh, sh, bh, nullptr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  p.d = (int)d; p.r = (int)r; p.T = (int)mid; p.b = (int)b;
}



// products one split accumulates in TMEM, at most (tc_conv.cu kCsumChain: the tensor core's fp32
// accumulation is not round-to-nearest, so chains stay short and the splits are added in fp32)
constexpr int64_t kChain = 512;
}  // namespace

// DPG_TG_LIN_BN=128: the rule on 128-wide double-buffered tiles only (A/B)
int lin_rule_bn() {
  static const int bn = [] {
    const char* e = std::getenv("DPG_TG_LIN_BN");
    return e && std::atoi(e) == 128 ? 128 : 256;
  }();
  return bn;
}

bool lin_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DPG_TG");
    const char* l = std::getenv("DPG_TG_LIN");
    return !(e && e[0] == '0') && !(l && l[0] == '0');
  }();
  return on;
}

bool lin_shape_ok(int64_t b, int64_t mid, int64_t d, int64_t r) {
  return lin_enabled() && b > 0 && mid > 1 && mid <= kChain && d % 4 == 0 && r % 4 == 0 && d >= 32 && r >= 32 &&
         b * mid * std::max(d, r) < (int64_t(1) << 31) && b * r * d < (int64_t(1) << 31);
}

bool lin_ok(const void* acts, const void* hw, const void* out, int64_t b, int64_t mid, int64_t d, int64_t r) {
  return lin_shape_ok(b, mid, d, r) && (reinterpret_cast<uintptr_t>(acts) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(hw) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
}

void lin_rule(dpg_ctx* ctx, const float* acts, int relu, const float* hw, int64_t b, int64_t mid, int64_t d,
              int64_t r, float* gw, double* sq_part) {
  const int mtiles = (int)((d + BM - 1) / BM);
  auto go = [&](auto BKc, auto BNc) {
    constexpr int BK = decltype(BKc)::value, BN = decltype(BNc)::value;
    using Pr = LinRuleT<BK, BN>;
    Pr p;
    set_maps<BK>(p, acts, hw, b, mid, d, r);
    p.relu = relu; p.sq = sq_part; p.mtiles = mtiles; p.nrows128 = (int)((r + 127) / 128);
    p.out = gw; p.stream = true;
    const unsigned ntiles = (unsigned)((r + BN - 1) / BN);
    launch<BN, BK, stages_for<BN, BK, stg_bytes<Pr>(), 0, 0, BN, Pr::kAccBufs>()>(ctx, p,
                                                                              dim3((unsigned)mtiles, ntiles, (unsigned)b));
  };
  const bool wide = r > 128 && lin_rule_bn() == 256;
  if (pick_bk(mid) == 16) {
    if (wide) go(std::integral_constant<int, 16>{}, std::integral_constant<int, 256>{});
    else go(std::integral_constant<int, 16>{}, std::integral_constant<int, 128>{});
  } else {
    if (wide) go(std::integral_constant<int, 32>{}, std::integral_constant<int, 256>{});
    else go(std::integral_constant<int, 32>{}, std::integral_constant<int, 128>{});
  }
}

// samples per split: chains <= kChain products; minimise (waves of the persistent grid x K blocks
// per tile) + the split-order reduce's partial traffic, both in K-block units (~0.42 us per
// 128 x 128 x 32 block at 3 MMAs per K slice; ~0.32 us per 2 MB of partials)
int lin_csum_splits(int64_t b, int64_t mid, int64_t d, int64_t r) {
  const int bk = pick_bk(mid);
  const int64_t kpt = (mid + bk - 1) / bk;
  const int64_t mn = ((d + BM - 1) / BM) * ((r + kLinBN - 1) / kLinBN);
  const int64_t spl_max = std::max<int64_t>(1, std::min<int64_t>(b, kChain / mid));
  double best = 1e300;
  int64_t best_spl = spl_max;
  for (int64_t spl = 1; spl <= spl_max; ++spl) {
    const int64_t splits = (b + spl - 1) / spl;
    const int64_t waves = (mn * splits + kNumSMs - 1) / kNumSMs;
    const double kblock_us = 0.42 * bk / 32.0 * (double)((std::min<int64_t>(d, BM) * std::min<int64_t>(r, kLinBN))) /
                             (double)(BM * kLinBN);
    const double cost = (double)(waves * spl * kpt) * kblock_us + (double)splits * (double)(d * r) * 8.0 / 6.5e6;
    if (cost < best) {
      best = cost;
      best_spl = spl;
    }
  }
  if (const char* e = std::getenv("DPG_TG_LIN_SPL")) best_spl = std::min<int64_t>(spl_max, std::max(1, std::atoi(e)));
  return (int)((b + best_spl - 1) / best_spl);
}

void lin_csum(dpg_ctx* ctx, const float* acts, int relu, const float* hw, const float* scale, int64_t b,
              int64_t mid, int64_t d, int64_t r, float* part, int splits) {
  const int mtiles = (int)((d + BM - 1) / BM), ntiles = (int)((r + kLinBN - 1) / kLinBN);
  auto go = [&](auto BKc) {
    constexpr int BK = decltype(BKc)::value;
    LinCsumT<BK> p;
    set_maps<BK>(p, acts, hw, b, mid, d, r);
    p.relu = relu; p.svec = scale;
    if constexpr (LinCsumT<BK>::kBRawMN) {
      const uint64_t dh[3] = {(uint64_t)r, (uint64_t)mid, (uint64_t)b};
      const uint64_t sh[2] = {(uint64_t)r * 4, (uint64_t)(mid * r * 4)};
      const uint32_t bh[3] = {(uint32_t)kLinBN, (uint32_t)BK, 1};
      p.mh = make_map(hw, 3, dh, sh, bh, nullptr, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
    p.out = part; p.stream = false;
    p.spl = (int)((b + splits - 1) / splits);
    p.kpt = (int)((mid + BK - 1) / BK);
    launch<kLinBN, BK, stages_for<kLinBN, BK, LinCsumT<BK>::kStaging>()>(ctx, p,
                                                                         dim3((unsigned)mtiles, (unsigned)ntiles, (unsigned)splits));
  };
  if (pick_bk(mid) == 16) go(std::integral_constant<int, 16>{});
  else go(std::integral_constant<int, 32>{});
}

}  // namespace tg
}  // namespace dpg

#ifdef DPG_TG_TRACE
// trace builds only (tools/tg_trace_lin.py): this translation unit's copy of the timeline
extern "C" __attribute__((visibility("default"))) void dpg_tg_lin_trace_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, dpg::tg::g_tg_trace, sizeof(unsigned long long) * 10 * 256);
}
#endif
