// cv_conv.cu — conv forward and conv input-gradient as one "direct conv on tensor cores" kernel.
//
// Both are a correlation of an input tensor X[n][ci][hin][win] with a tap window:
//   out[(n, qy, qx)][co] = sum_{ci, ty, tx} X[n][ci][qy*sq + oy + ty][qx*sq + ox + tx] * Wk[co][ci][ty][tx]
//   forward (layers.hpp:432-467):  X = x (ReLU on load), sq = stride, (oy, ox) = -pad, Wk = W,
//                                  out -> y[n][co][qy*ow + qx] + bias
//   dgrad   (layers.hpp:630-649 + col2im :326-358), per stride-parity class (ry, rx) of input
//           pixels: X = dy, sq = 1, the class's taps ki = ry + s a, kj = rx + s c read dy at
//           (oy0 - a, ox0 - c); flipping the tap order (ty = nki-1-a) makes it a forward
//           correlation with origin oy0 - (nki-1); out -> dx[n][c][iy0 + s qy][ix0 + s qx],
//           masked by the producing layer's ReLU (layers.hpp:712-718).
//
// GEMM view: rows = output positions (UMMA M = 128 = TMEM lanes = epilogue threads, contiguous in
// the output), columns = output channels (UMMA N), K = (channel group, channel, tap) with
// cps = floor(32 / taps) channels per 32-wide K stage (zero padded), so every stage needs exactly
// cps channels of the CTA's samples. Per stage:
//   * cp.async (16 B) stages those channel planes of the CTA's samples into shared memory (raw
//     fp32) one stage ahead;
//   * the weights were pre-packed once per step (pack_weights_kernel) into per-(stage, column
//     tile) TF32 hi / lo 128B-swizzled K-major tiles, copied straight into the B operand buffers;
//   * the threads build the A tile (hi / lo, swizzled) from the staged planes;
//   * one thread issues 3 x 4 tcgen05.mma.kind::tf32 (lo*hi + hi*lo + hi*hi per K=8 slice) into
//     the TMEM accumulator and commits to the stage's mbarrier.
#include <cstdlib>

#include "conv_common.cuh"
#include "tc_gemm.cuh"

namespace dpg {
namespace cv {

using tc::BK;
using tc::BM;
constexpr int kThreads = 256;

struct Conv {
  // input
  const float* x;
  int relu;
  int ci, hin, win;
  // output grid / window
  int hq, wq, sq, oy, ox;
  int th, tw, cps, nstages;
  int co;  // output channels (GEMM N)
  // packed weights [nstages][ntiles][2][BN][32]
  const float* wpack;
  int64_t M;  // b * hq * wq
  int spc;    // samples per CTA tile (ceil(128 / (hq*wq)) + 1 upper bound)
  int raw_floats;  // per stage buffer
  // epilogue
  int mode;  // 0 = forward, 1 = dgrad
  float* y;
  const float* bias;
  float* dx;
  const float* mask;
  int dh, dw, dci, iy0, ix0, ds;  // dgrad output geometry: dx [n][dci][dh][dw], pixel (iy0 + ds qy, ix0 + ds qx)
  int ksplit;
  float* part;  // split-K partials [ksplit][co][M]
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Pipeline (stage = 32-wide K slice; a 12-MMA 3xTF32 stage takes ~1000 cycles on the tensor
// pipe, measured): copies run 2 stages ahead (raw planes ring of 3, packed-weight ring of 4), the A
// tile is double buffered, so MMA(i-1) executes while the threads build A(i) and the only wait is
// on MMA(i-2).
constexpr int kRing = 3;   // raw-plane ring
constexpr int kWRing = 4;  // packed-weight ring (slot i+2 reuses the slot MMA(i-2) read)

template <int BN>
struct CvSmem {
  static constexpr int A_BYTES = BM * BK * 4;          // 16 KB per hi / lo
  static constexpr int W_BYTES = 2 * BN * BK * 4;      // packed hi + lo tile
  static constexpr int A_REGION = 2 * 2 * A_BYTES;     // two buffers x (hi, lo)
  static constexpr int W_REGION = kWRing * W_BYTES;
  static constexpr int FIXED = A_REGION + W_REGION + 64;
};

template <int BN>
__global__ void __launch_bounds__(kThreads) conv_tc_kernel(const Conv p) {
  using S = CvSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  // 1024 B alignment by pointer arithmetic on the __shared__ array, so the compiler keeps the
  // shared address space (LDS / STS, not generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  uint8_t* abuf = smem;                                // [2][hi | lo]
  uint8_t* wring = smem + S::A_REGION;                 // [kWRing][hi | lo] packed tiles (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::A_REGION + S::W_REGION);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  float* raw = reinterpret_cast<float*>(smem + S::FIXED);  // [kRing][raw_floats]

  const int tid = threadIdx.x, warp = tid >> 5;
  const int split = blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  constexpr uint32_t kCols = tc::tmem_cols<BN>();
  const int pq = p.hq * p.wq;
  const int nbase = (int)(m0 / pq);  // first sample of the tile
  const int hw_in = p.hin * p.win;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // This thread's A row and k quads never change across stages (the tap pattern of every stage
  // is the same: cps channels x taps), so its 16 shared-memory offsets and validity bits are
  // computed once here.
  const int row = tid & 127;
  const int64_t m = m0 + row;
  int offs[16];
  uint32_t valid = 0;
  {
    int rs = 0, ry0 = -(1 << 14), rx0 = -(1 << 14);
    if (m < p.M) {
      const int n = (int)(m / pq), q = (int)(m - (int64_t)n * pq);
      const int qy = q / p.wq, qx = q - qy * p.wq;
      rs = n - nbase;
      ry0 = qy * p.sq + p.oy;
      rx0 = qx * p.sq + p.ox;
    }
    const int taps = p.th * p.tw;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = 4 * ((tid >> 7) + 2 * j) + e;
        int off = 0;
        if (k < p.cps * taps) {
          const int cl = k / taps, t = k - cl * taps;
          const int yy = ry0 + t / p.tw, xx = rx0 + t % p.tw;
          if ((unsigned)yy < (unsigned)p.hin && (unsigned)xx < (unsigned)p.win) {
            off = ((rs * p.cps + cl) * p.hin + yy) * p.win + xx;
            valid |= 1u << (4 * j + e);
          }
        }
        offs[4 * j + e] = off;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int ks0 = (int)((int64_t)split * p.nstages / p.ksplit);
  const int ks1 = (int)((int64_t)(split + 1) * p.nstages / p.ksplit);
  const int nk = ks1 - ks0;
  const int64_t last_m = (m0 + BM < p.M ? m0 + BM : p.M) - 1;
  const int nsamp = (int)(last_m / pq) - nbase + 1;

  // issue the copies of local stage i (channel planes + packed weights) into ring slot i % kRing;
  // channels past ci (last stage) are zero-filled so the precomputed offsets stay valid
  auto issue = [&](int i) {
    const int slot = i % kRing, wslot = i % kWRing;
    const int st = ks0 + i;
    float* dst = raw + slot * p.raw_floats;
    const int c0 = st * p.cps;
    const int nc = min(p.cps, p.ci - c0);
    if ((hw_in & 3) == 0) {
      const int q4 = hw_in >> 2;
      const int total = nsamp * nc * q4;
      for (int k = tid; k < total; k += kThreads) {
        const int plane = k / q4, j = k - plane * q4;
        const int sl = plane / nc, cl = plane - sl * nc;
        cp_async16(dst + (sl * p.cps + cl) * hw_in + 4 * j,
                   p.x + ((int64_t)(nbase + sl) * p.ci + c0 + cl) * hw_in + 4 * j);
      }
    } else {
      const int total = nsamp * nc * hw_in;
      for (int k = tid; k < total; k += kThreads) {
        const int plane = k / hw_in, j = k - plane * hw_in;
        const int sl = plane / nc, cl = plane - sl * nc;
        cp_async4(dst + (sl * p.cps + cl) * hw_in + j, p.x + ((int64_t)(nbase + sl) * p.ci + c0 + cl) * hw_in + j);
      }
    }
    if (nc < p.cps) {
      const int missing = (p.cps - nc) * hw_in;
      for (int k = tid; k < nsamp * missing; k += kThreads) {
        const int sl = k / missing, j = k - sl * missing;
        dst[(sl * p.cps + nc) * hw_in + j] = 0.f;
      }
    }
    const float* wsrc = p.wpack + ((int64_t)st * gridDim.y + blockIdx.y) * (2 * BN * BK);
    uint8_t* wdst = wring + wslot * S::W_BYTES;
    constexpr int chunks = 2 * BN * BK / 4;
    for (int k = tid; k < chunks; k += kThreads) cp_async16(wdst + 16 * k, wsrc + 4 * k);
  };

  if (nk > 0) issue(0);
  cp_commit();
  if (nk > 1) issue(1);
  cp_commit();
  constexpr uint32_t idesc = tc::idesc_tf32(BN);
  for (int i = 0; i < nk; ++i) {
    const int slot = i % kRing, wslot = i % kWRing, ab = i & 1;
    cp_wait<1>();  // stage i landed (stage i + 1 may still be in flight)
    __syncthreads();
    // MMA(i - 2) done: A[ab] and weight slot (i + 2) % kWRing are free; MMA(i - 1) may still run
    if (i >= 2) tc::mbar_wait(&bars[ab], ((i >> 1) - 1) & 1);
    if (i + 2 < nk) issue(i + 2);
    cp_commit();
    uint8_t* a_hi = abuf + ab * 2 * S::A_BYTES;
    uint8_t* a_lo = a_hi + S::A_BYTES;
    const float* rb = raw + slot * p.raw_floats;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = 4 * j + e;
        const float x = rb[offs[idx]];
        v[e] = (valid >> idx) & 1 ? relu_if(x, p.relu) : 0.f;
      }
      tc::put4(a_hi, a_lo, row, (tid >> 7) + 2 * j, v[0], v[1], v[2], v[3]);
    }
    tc::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
      const uint32_t sa_hi = tc::smem_u32(a_hi), sa_lo = tc::smem_u32(a_lo);
      const uint32_t sb_hi = tc::smem_u32(wring + wslot * S::W_BYTES);
      const uint32_t sb_lo = sb_hi + BN * BK * 4;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint32_t off = kk * 32;
        const uint32_t acc0 = (i > 0 || kk > 0) ? 1u : 0u;
        tc::mma_tf32(tmem, tc::sw128_desc(sa_lo + off), tc::sw128_desc(sb_hi + off), idesc, acc0);
        tc::mma_tf32(tmem, tc::sw128_desc(sa_hi + off), tc::sw128_desc(sb_lo + off), idesc, 1u);
        tc::mma_tf32(tmem, tc::sw128_desc(sa_hi + off), tc::sw128_desc(sb_hi + off), idesc, 1u);
      }
      tc::mma_commit(&bars[ab]);
    }
  }
  if (nk > 0) tc::mbar_wait(&bars[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
  tc::tc_fence_after();

  // epilogue: warp w -> TMEM lanes [32 (w % 4), +32), column half w / 4
  const int lane_base = 32 * (warp & 3);
  const int64_t me = m0 + lane_base + (tid & 31);
  const bool row_ok = me < p.M;
  constexpr int HALF = BN / 2 >= 16 ? BN / 2 : 16;
  const int c_begin = (warp >> 2) * HALF;
  int en = 0, eqy = 0, eqx = 0;
  if (row_ok) {
    en = (int)(me / pq);
    const int q = (int)(me - (int64_t)en * pq);
    eqy = q / p.wq;
    eqx = q - eqy * p.wq;
  }
  float v[16];
  if (c_begin < BN) {
#pragma unroll 1
    for (int c0 = c_begin; c0 < c_begin + HALF && c0 < BN; c0 += 16) {
      if (nk > 0) {
        tc::tmem_ld16(tmem + ((uint32_t)lane_base << 16) + (uint32_t)c0, v);
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = 0.f;
      }
      if (!row_ok) continue;
      const int nv = min(16, p.co - (n0 + c0));
      if (p.ksplit > 1) {
        float* out = p.part + ((int64_t)split * p.co + n0 + c0) * p.M + me;
        #pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < nv) out[(int64_t)j * p.M] = v[j];
      } else if (p.mode == 0) {
        float* out = p.y + ((int64_t)en * p.co + n0 + c0) * pq + eqy * p.wq + eqx;
        #pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < nv) out[(int64_t)j * pq] = v[j] + (p.bias ? __ldg(p.bias + n0 + c0 + j) : 0.f);
      } else {
        const int64_t hw = (int64_t)p.dh * p.dw;
        const int64_t off0 = ((int64_t)en * p.dci + n0 + c0) * hw + (int64_t)(p.iy0 + p.ds * eqy) * p.dw + p.ix0 + p.ds * eqx;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j >= nv) continue;
          const int64_t off = off0 + (int64_t)j * hw;
          float val = v[j];
          if (p.mask && !(__ldg(p.mask + off) > 0.f)) val = 0.f;
          p.dx[off] = val;
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
  }
}

// ---------------------------------------------------------------------------------------------
// Weight packing: Wk[co][k] with k = (stage, c_local, tap) -> per (stage, column tile) the TF32 hi
// and lo 128B-swizzled K-major tiles [2][BN][32] the kernel copies straight into its B buffers.
// wsrc(co, ci, ty, tx) is the tap weight in the kernel's (flipped for dgrad) order.
struct WSrc {
  const float* w;  // reference layout [oc][ic][kh][kw]
  int oc, ic, kh, kw;
  int dgrad;       // 0: forward (co = oc, ci = ic); 1: dgrad class (co = ic, ci = oc)
  int ry, rx, s, nki, nkj;
  __device__ float operator()(int co, int ci, int ty, int tx) const {
    if (!dgrad) return __ldg(w + (((int64_t)co * ic + ci) * kh + ty) * kw + tx);
    const int a = nki - 1 - ty, c = nkj - 1 - tx;  // flipped tap order
    return __ldg(w + (((int64_t)ci * ic + co) * kh + ry + s * a) * kw + rx + s * c);
  }
};

__global__ void pack_weights_kernel(WSrc src, int co_n, int ci_n, int th, int tw, int cps, int nstages,
                                    int bn, int ntiles, float* out) {
  const int64_t total = (int64_t)nstages * ntiles * bn * BK;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int k = (int)(i % BK);
  const int r = (int)((i / BK) % bn);
  const int tile = (int)((i / ((int64_t)BK * bn)) % ntiles);
  const int st = (int)(i / ((int64_t)BK * bn * ntiles));
  const int taps = th * tw;
  const int co = tile * bn + r;
  float v = 0.f;
  if (k < cps * taps && co < co_n) {
    const int cl = k / taps, t = k - cl * taps;
    const int ci = st * cps + cl;
    if (ci < ci_n) v = src(co, ci, t / tw, t % tw);
  }
  const uint32_t hi = tc::to_tf32(v);
  const uint32_t lo = tc::to_tf32(v - __uint_as_float(hi));
  // swizzled byte offset of (row r, element k) inside a [bn][32] SW128 tile
  const uint32_t off = tc::sw128_off(r, k >> 2) + (k & 3) * 4;
  uint8_t* base = reinterpret_cast<uint8_t*>(out + ((int64_t)st * ntiles + tile) * 2 * bn * BK);
  *reinterpret_cast<uint32_t*>(base + off) = hi;
  *reinterpret_cast<uint32_t*>(base + (size_t)bn * BK * 4 + off) = lo;
}

// ---------------------------------------------------------------------------------------------
static int pick_bn(int n) { return n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : 128; }

struct Plan {
  int bn, ntiles, cps, nstages, taps, spc, raw_floats, ksplit;
  int64_t M;
  size_t pack_floats, part_floats, smem;
};

static Plan plan(int64_t b, int ci, int hin, int win, int hq, int wq, int th, int tw, int co,
                 bool allow_split, int64_t grid_z_extra = 1) {
  Plan pl{};
  pl.taps = th * tw;
  pl.cps = BK / pl.taps;
  pl.bn = pick_bn(co);
  pl.ntiles = (co + pl.bn - 1) / pl.bn;
  pl.nstages = pl.cps > 0 ? (ci + pl.cps - 1) / pl.cps : 0;
  pl.M = b * hq * wq;
  const int pq = hq * wq;
  // samples a 128-row tile can span (tiles start at multiples of 128)
  pl.spc = (pq % BM == 0) ? 1 : (BM % pq == 0) ? BM / pq : (BM + pq - 1) / pq + 1;
  pl.raw_floats = ((pl.spc * pl.cps * hin * win) + 3) & ~3;
  pl.pack_floats = (size_t)pl.nstages * pl.ntiles * 2 * pl.bn * BK;
  const int64_t tiles = ((pl.M + BM - 1) / BM) * pl.ntiles * grid_z_extra;
  pl.ksplit = 1;
  if (allow_split && tiles < kNumSMs) {
    pl.ksplit = (int)std::min<int64_t>(std::max<int64_t>(1, pl.nstages / 2), (2 * kNumSMs + tiles - 1) / tiles);
    pl.ksplit = std::max(1, std::min(pl.ksplit, 16));
  }
  pl.part_floats = pl.ksplit > 1 ? (size_t)pl.ksplit * co * pl.M : 0;
  const int sfix = pl.bn == 16 ? CvSmem<16>::FIXED : pl.bn == 32 ? CvSmem<32>::FIXED
                 : pl.bn == 64 ? CvSmem<64>::FIXED : CvSmem<128>::FIXED;
  pl.smem = (size_t)sfix + 1024 + sizeof(float) * kRing * pl.raw_floats;
  return pl;
}

static bool plan_ok(const Plan& pl) { return pl.cps > 0 && pl.smem <= 220 * 1024; }

template <int BN>
static void launch_bn(dpg_ctx* ctx, const Conv& p, const Plan& pl) {
  static size_t attr = 0;
  if (pl.smem > attr) {
    DPG_CUDA(cudaFuncSetAttribute(conv_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    attr = pl.smem;
  }
  dim3 grid((unsigned)((p.M + BM - 1) / BM), (unsigned)pl.ntiles, (unsigned)p.ksplit);
  conv_tc_kernel<BN><<<grid, kThreads, pl.smem, ctx->stream>>>(p);
  DPG_LAUNCH_CHECK(ctx);
}

static void launch(dpg_ctx* ctx, const Conv& p, const Plan& pl) {
  switch (pl.bn) {
    case 16: launch_bn<16>(ctx, p, pl); break;
    case 32: launch_bn<32>(ctx, p, pl); break;
    case 64: launch_bn<64>(ctx, p, pl); break;
    default: launch_bn<128>(ctx, p, pl); break;
  }
}

static void pack(dpg_ctx* ctx, const WSrc& src, int co, int ci, int th, int tw, const Plan& pl, float* out) {
  const int64_t total = (int64_t)pl.nstages * pl.ntiles * pl.bn * BK;
  pack_weights_kernel<<<(unsigned)((total + 255) / 256), 256, 0, ctx->stream>>>(src, co, ci, th, tw, pl.cps,
                                                                                 pl.nstages, pl.bn, pl.ntiles, out);
  DPG_LAUNCH_CHECK(ctx);
}

bool enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DPG_CV");
    return e && e[0] == '1';  // opt-in: measured slower than the gather path
  }();
  return on;
}

// ---- forward ----
static Plan fwd_plan(const ConvGeom& g) {
  return plan(g.b, (int)g.ic, (int)g.h, (int)g.w, (int)g.oh, (int)g.ow, (int)g.kh, (int)g.kw, (int)g.oc, true);
}
bool fwd_supported(const ConvGeom& g) { return enabled() && plan_ok(fwd_plan(g)); }
size_t fwd_ws_bytes(const ConvGeom& g) {
  const Plan pl = fwd_plan(g);
  return sizeof(float) * (pl.pack_floats + pl.part_floats) + 256;
}

__global__ void fwd_reduce_kernel(const float* __restrict__ part, int ksplit, int64_t M, int co, int P,
                                  const float* __restrict__ bias, float* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)co * M) return;
  const int64_t c = i / M, m = i - c * M;
  float acc = 0.f;
  for (int s = 0; s < ksplit; ++s) acc += part[(int64_t)s * co * M + i];
  const int64_t n = m / P, q = m - n * P;
  y[(n * co + c) * P + q] = acc + (bias ? bias[c] : 0.f);
}

void conv_fwd(dpg_ctx* ctx, const float* x, int relu, const float* w, const float* bias, const ConvGeom& g,
              float* y, void* ws) {
  const Plan pl = fwd_plan(g);
  float* wpack = static_cast<float*>(ws);
  float* part = wpack + pl.pack_floats;
  WSrc src{w, (int)g.oc, (int)g.ic, (int)g.kh, (int)g.kw, 0, 0, 0, 1, 0, 0};
  pack(ctx, src, (int)g.oc, (int)g.ic, (int)g.kh, (int)g.kw, pl, wpack);
  Conv p{};
  p.x = x; p.relu = relu; p.ci = (int)g.ic; p.hin = (int)g.h; p.win = (int)g.w;
  p.hq = (int)g.oh; p.wq = (int)g.ow; p.sq = (int)g.stride; p.oy = -(int)g.pad; p.ox = -(int)g.pad;
  p.th = (int)g.kh; p.tw = (int)g.kw; p.cps = pl.cps; p.nstages = pl.nstages; p.co = (int)g.oc;
  p.wpack = wpack; p.M = pl.M; p.spc = pl.spc; p.raw_floats = pl.raw_floats;
  p.mode = 0; p.y = y; p.bias = bias;
  p.ksplit = pl.ksplit; p.part = part;
  launch(ctx, p, pl);
  if (pl.ksplit > 1) {
    const int64_t n = (int64_t)g.oc * pl.M;
    fwd_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(part, pl.ksplit, pl.M, (int)g.oc,
                                                                             (int)g.P(), bias, y);
    DPG_LAUNCH_CHECK(ctx);
  }
}

// ---- dgrad: one launch per stride-parity class ----
struct DClass {
  int ry, rx, iy0, ix0, hc, wc, nki, nkj;
};
static DClass dclass(const ConvGeom& g, int ry, int rx) {
  const int s = (int)g.stride;
  DClass c{};
  c.ry = ry; c.rx = rx;
  c.iy0 = ((ry - (int)g.pad) % s + s) % s;
  c.ix0 = ((rx - (int)g.pad) % s + s) % s;
  c.hc = c.iy0 < g.h ? (int)((g.h - c.iy0 + s - 1) / s) : 0;
  c.wc = c.ix0 < g.w ? (int)((g.w - c.ix0 + s - 1) / s) : 0;
  c.nki = ry < g.kh ? (int)((g.kh - ry + s - 1) / s) : 0;
  c.nkj = rx < g.kw ? (int)((g.kw - rx + s - 1) / s) : 0;
  return c;
}
static Plan dgrad_plan(const ConvGeom& g, const DClass& c) {
  return plan(g.b, (int)g.oc, (int)g.oh, (int)g.ow, c.hc, c.wc, std::max(1, c.nki), std::max(1, c.nkj),
              (int)g.ic, true);
}
bool dgrad_supported(const ConvGeom& g) {
  if (!enabled()) return false;
  const int s = (int)g.stride;
  for (int ry = 0; ry < s; ++ry)
    for (int rx = 0; rx < s; ++rx) {
      const DClass c = dclass(g, ry, rx);
      if (c.hc == 0 || c.wc == 0) continue;
      if (!plan_ok(dgrad_plan(g, c))) return false;
    }
  return true;
}
size_t dgrad_ws_bytes(const ConvGeom& g) {
  size_t best = 0;
  const int s = (int)g.stride;
  for (int ry = 0; ry < s; ++ry)
    for (int rx = 0; rx < s; ++rx) {
      const DClass c = dclass(g, ry, rx);
      if (c.hc == 0 || c.wc == 0) continue;
      const Plan pl = dgrad_plan(g, c);
      best = std::max(best, sizeof(float) * (pl.pack_floats + pl.part_floats) + 256);
    }
  return best;
}

__global__ void dgrad_reduce_kernel(const float* __restrict__ part, int ksplit, int64_t M, int co,
                                    int hc, int wc, int h, int w, int iy0, int ix0, int s,
                                    const float* __restrict__ mask, float* __restrict__ dx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)co * M) return;
  const int64_t c = i / M, m = i - c * M;
  float acc = 0.f;
  for (int k = 0; k < ksplit; ++k) acc += part[(int64_t)k * co * M + i];
  const int pq = hc * wc;
  const int64_t n = m / pq;
  const int q = (int)(m - n * pq), qy = q / wc, qx = q - qy * wc;
  const int64_t off = ((n * co + c) * h + iy0 + s * qy) * (int64_t)w + ix0 + s * qx;
  if (mask && !(mask[off] > 0.f)) acc = 0.f;
  dx[off] = acc;
}

void conv_dgrad(dpg_ctx* ctx, const float* dy, const float* w, const ConvGeom& g, const float* mask,
                float* dx, void* ws) {
  const int s = (int)g.stride;
  for (int ry = 0; ry < s; ++ry)
    for (int rx = 0; rx < s; ++rx) {
      const DClass c = dclass(g, ry, rx);
      if (c.hc == 0 || c.wc == 0) continue;
      if (c.nki == 0 || c.nkj == 0) {
        // no tap reaches this class: its input gradient is exactly zero
        raise(DPG_ERR_INTERNAL, "dgrad class without taps (kernel smaller than stride) unsupported on cv path");
      }
      const Plan pl = dgrad_plan(g, c);
      float* wpack = static_cast<float*>(ws);
      float* part = wpack + pl.pack_floats;
      WSrc src{w, (int)g.oc, (int)g.ic, (int)g.kh, (int)g.kw, 1, c.ry, c.rx, s, c.nki, c.nkj};
      pack(ctx, src, (int)g.ic, (int)g.oc, c.nki, c.nkj, pl, wpack);
      Conv p{};
      p.x = dy; p.relu = 0; p.ci = (int)g.oc; p.hin = (int)g.oh; p.win = (int)g.ow;
      p.hq = c.hc; p.wq = c.wc; p.sq = 1;
      // input pixel (iy0 + s qy) reads dy at oy0 - a with oy0 = (iy + pad - ry) / s; flipped tap
      // ty = nki - 1 - a  ->  window origin oy0 - (nki - 1) = qy + (iy0 + pad - ry) / s - (nki - 1)
      p.oy = (c.iy0 + (int)g.pad - c.ry) / s - (c.nki - 1);
      p.ox = (c.ix0 + (int)g.pad - c.rx) / s - (c.nkj - 1);
      p.th = c.nki; p.tw = c.nkj; p.cps = pl.cps; p.nstages = pl.nstages; p.co = (int)g.ic;
      p.wpack = wpack; p.M = pl.M; p.spc = pl.spc; p.raw_floats = pl.raw_floats;
      p.mode = 1; p.dx = dx; p.mask = mask;
      p.dh = (int)g.h; p.dw = (int)g.w; p.dci = (int)g.ic; p.iy0 = c.iy0; p.ix0 = c.ix0; p.ds = s;
      p.ksplit = pl.ksplit; p.part = part;
      launch(ctx, p, pl);
      if (pl.ksplit > 1) {
        const int64_t n = (int64_t)g.ic * pl.M;
        dgrad_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
            part, pl.ksplit, pl.M, (int)g.ic, c.hc, c.wc, (int)g.h, (int)g.w, c.iy0, c.ix0, s, mask, dx);
        DPG_LAUNCH_CHECK(ctx);
      }
    }
}

}  // namespace cv
}  // namespace dpg
