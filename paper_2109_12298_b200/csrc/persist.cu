// persist.cu — the whole DP-SGD step of a small model in ONE cooperative kernel (SURVEY.md §8f
// row 3: "a persistent single-kernel step for small batches").
//
// A small batch (MNIST CNN, b = 64: 26,010 parameters, 6.7 MB of per-sample gradients) is bound
// by launch latency, not by the GPU: the multi-kernel step is 22 launches at ~3 µs each. Here one
// grid (every SM, co-resident by cooperative launch) walks the reference's step; only the phases
// that combine samples are separated by grid barriers (three):
//
//   per sample, in one CTA, every activation and highway in shared memory (no grid barrier):
//     forward(l)          layer_forward, layers.hpp:389-413 (linear), :432-467 (conv2d), ReLU
//                         applied on load
//     loss                softmax-CE in double (layers.hpp:894-919)
//     backward(l), L..1   per_sample_rule_{linear,conv2d} (grad_sample.hpp:53-59, 135-150) into the
//                         record with the bias rule's sequential double sum (sum_middle,
//                         tensor.hpp:188-207), backward_input with the ReLU mask (layers.hpp:606-649,
//                         712-718), and clip_and_sum pass 1 (optimizer.hpp:67-89): per (parameter,
//                         sample) double sums, first non-finite (l, k, n) reported as the NumericError
//   factors               optimizer.hpp:90-98
//   clipped sum           optimizer.hpp:99-114 from the record, in the reference's own order (n
//                         ascending, fp32 multiply then add): bit-exact given the record
//   noise + update        the multi-kernel step's Philox stream and two-rounding update
//                         (optimizer.hpp:120-133, 256-271), skipped when an error is pending
//
// Scope (persist_ok): conv2d (groups of 1) / linear (one row per sample) / relu / flatten models,
// the record materialised, one GPU, a fresh logical batch (dpg_train_step). Everything else takes
// the multi-kernel step. Reads of data written by other CTAs earlier in the kernel bypass L1
// (__ldcg): L1 is not coherent across SMs.
#include <algorithm>

#include "persist.h"
#include "step_common.cuh"

namespace dpg {
namespace ps {

#ifdef DPG_PERSIST_TRACE
__device__ unsigned long long g_persist_trace[32];  // CTA 0's globaltimer at each barrier
__device__ int g_persist_ev;
#endif

// sense-reversing grid barrier (all CTAs co-resident: cooperative launch)
__device__ __forceinline__ void grid_sync(unsigned int* bar) {
#ifdef DPG_PERSIST_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_persist_trace[g_persist_ev++ & 31] = t;
  }
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

// ---- phase A: one sample per CTA, every intermediate in shared memory ----
// forward of layer l: out = bias + sum W x~ (pre-activation), input ReLU applied on load
__device__ void forward(const PLayer l, float* sm) {  // by value: the fields live in registers
  const float* in = sm + l.in_s;
  float* out = sm + l.out_s;
  if (l.conv) {
    const int P = l.OH * l.OW;
    for (int j = threadIdx.x; j < l.O * P; j += kThreads) {
      const int o = j / P, p = j - o * P;
      const int oy = p / l.OW, ox = p - oy * l.OW;
      const float* wo = l.w + (int64_t)o * l.C * l.KH * l.KW;
      float acc = 0.f;
      for (int c = 0; c < l.C; ++c)
        for (int ki = 0; ki < l.KH; ++ki) {
          const int iy = oy * l.S - l.PAD + ki;
          if ((unsigned)iy >= (unsigned)l.H) continue;
          const float* xr = in + (c * l.H + iy) * l.W;
          const float* wr = wo + (c * l.KH + ki) * l.KW;
          for (int kj = 0; kj < l.KW; ++kj) {
            const int ix = ox * l.S - l.PAD + kj;
            if ((unsigned)ix < (unsigned)l.W) acc = fmaf(__ldg(wr + kj), relu_if(xr[ix], l.in_relu), acc);
          }
        }
      out[j] = acc + (l.bias ? __ldg(l.bias + o) : 0.f);
    }
  } else {  // a warp per output, lanes across the inputs, fixed shuffle tree
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < l.O; j += kThreads / 32) {
      const float* wo = l.w + (int64_t)j * l.C;
      float acc = 0.f;
      for (int i = lane; i < l.C; i += 32) acc = fmaf(__ldg(wo + i), relu_if(in[i], l.in_relu), acc);
      acc = warp_sum(acc);
      if (lane == 0) out[j] = acc + (l.bias ? __ldg(l.bias + j) : 0.f);
    }
  }
}

// backward of layer l for sample n: weight rule + bias rule into the record (with their squared
// norms) and the input gradient into the previous layer's highway (ReLU mask folded in)
__device__ void backward(const PLayer l, float* sm, int64_t n, double& sqw, double& sqb, int& badw, int& badb) {
  const float* in = sm + l.in_s;
  const float* hs = sm + l.hw_s;
  const int P = l.conv ? l.OH * l.OW : 1;
  float* gw = l.gw + n * l.numel_w;
  for (int64_t e = threadIdx.x; e < l.numel_w; e += kThreads) {
    float acc;
    if (l.conv) {  // G[o][k] = sum_p hw[o][p] x~[k][p], positions in order p = oy OW + ox
      const int K = l.C * l.KH * l.KW, o = (int)(e / K), k = (int)(e - (int64_t)o * K);
      const int c = k / (l.KH * l.KW), t = k - c * (l.KH * l.KW), ki = t / l.KW, kj = t - ki * l.KW;
      const float* ho = hs + o * P;
      const float* xc = in + c * l.H * l.W;
      acc = 0.f;
      for (int oy = 0; oy < l.OH; ++oy) {
        const int iy = oy * l.S - l.PAD + ki;
        const bool rowok = (unsigned)iy < (unsigned)l.H;
        for (int ox = 0; ox < l.OW; ++ox) {
          const int ix = ox * l.S - l.PAD + kj;
          const float xv = (rowok && (unsigned)ix < (unsigned)l.W) ? relu_if(xc[iy * l.W + ix], l.in_relu) : 0.f;
          acc = fmaf(ho[oy * l.OW + ox], xv, acc);
        }
      }
    } else {  // one product: bit-exact
      const int o = (int)(e / l.C), i = (int)(e - (int64_t)o * l.C);
      acc = hs[o] * relu_if(in[i], l.in_relu);
    }
    st_stream(gw + e, acc);
    badw |= !isfinite(acc);
    sqw += (double)acc * acc;
  }
  if (l.gb) {  // gb[o] = (float) sum_p (double) hw[o][p], p ascending
    for (int o = threadIdx.x; o < l.O; o += kThreads) {
      double a = 0.0;
      for (int pp = 0; pp < P; ++pp) a += (double)hs[o * P + pp];
      const float v = (float)a;
      l.gb[n * l.O + o] = v;
      badb |= !isfinite(v);
      sqb += (double)v * v;
    }
  }
  if (l.hw_prev_s < 0) return;
  float* hp = sm + l.hw_prev_s;
  for (int j = threadIdx.x; j < l.in_numel; j += kThreads) {
    float acc = 0.f;
    if (l.conv) {
      const int hwsz = l.H * l.W, c = j / hwsz, r = j - c * hwsz;
      const int iy = r / l.W, ix = r - iy * l.W;
      // only the taps that reach this pixel: ki = (iy + pad) mod s, + s, ... (oy = (iy + pad - ki) / s)
      const int ki0 = (iy + l.PAD) % l.S, kj0 = (ix + l.PAD) % l.S;
      const int64_t ostr = (int64_t)l.C * l.KH * l.KW;
      for (int ki = ki0; ki < l.KH; ki += l.S) {
        const int oy = (iy + l.PAD - ki) / l.S;
        if (oy >= l.OH) continue;
        if (oy < 0) break;
        for (int kj = kj0; kj < l.KW; kj += l.S) {
          const int ox = (ix + l.PAD - kj) / l.S;
          if (ox >= l.OW) continue;
          if (ox < 0) break;
          const float* wk = l.w + ((int64_t)c * l.KH + ki) * l.KW + kj;
          const float* ht = hs + oy * l.OW + ox;
          for (int o = 0; o < l.O; ++o) acc = fmaf(ht[o * P], __ldg(wk + o * ostr), acc);
        }
      }
    } else {
      for (int o = 0; o < l.O; ++o) acc = fmaf(hs[o], __ldg(l.w + (int64_t)o * l.C + j), acc);
    }
    if (l.in_relu && !(in[j] > 0.f)) acc = 0.f;  // the previous layer's ReLU
    hp[j] = acc;
  }
}

__device__ void sample_phase(const Params& p, float* sm) {
  __shared__ double red[kThreads / 32];
  __shared__ int flags[2];
  for (int64_t n = blockIdx.x; n < p.b; n += gridDim.x) {
    const PLayer& l0 = p.L[0];
    for (int64_t i = threadIdx.x; i < l0.in_numel; i += kThreads) sm[l0.in_s + i] = __ldg(l0.in + n * l0.in_numel + i);
    __syncthreads();
    for (int l = 0; l < p.nl; ++l) {
      forward(p.L[l], sm);
      __syncthreads();
    }
    const PLayer& lt = p.L[p.nl - 1];
    const int k = (int)lt.out_numel;
    if (threadIdx.x < 32)  // grad[n k + j] addresses the sample's highway row in shared memory
      softmax_ce_warp(sm + lt.out_s, p.out_relu, p.targets, n, k, p.loss, sm + lt.hw_s - n * k, p.err);
    __syncthreads();
    for (int l = p.nl - 1; l >= 0; --l) {
      const PLayer& L = p.L[l];
      double sqw = 0.0, sqb = 0.0;
      int badw = 0, badb = 0;
      if (threadIdx.x == 0) flags[0] = flags[1] = 0;
      __syncthreads();
      backward(L, sm, n, sqw, sqb, badw, badb);
      if (badw) flags[0] = 1;
      if (badb) flags[1] = 1;
      const double tw = block_sum<kThreads>(sqw, red);
      const double tb = L.gb ? block_sum<kThreads>(sqb, red) : 0.0;
      if (threadIdx.x == 0) {  // clip_and_sum pass 1 partials; first non-finite (l, k, n) wins
        p.part[(int64_t)L.pw * p.b + n] = tw;
        if (flags[0]) report_error(p.err, err_key(ERR_STAGE_NONFINITE, (uint64_t)L.pw, (uint64_t)n), 0);
        if (L.gb) {
          p.part[(int64_t)(L.pw + 1) * p.b + n] = tb;
          if (flags[1]) report_error(p.err, err_key(ERR_STAGE_NONFINITE, (uint64_t)(L.pw + 1), (uint64_t)n), 0);
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kThreads) persist_step_kernel(const __grid_constant__ Params p) {
  extern __shared__ float sm[];
  const uint64_t step = p.step_ptr ? *p.step_ptr : p.step;
  if (gtid() == 0 && p.num_clipped) *p.num_clipped = 0;
#ifdef DPG_PERSIST_TRACE
  if (gtid() == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ps::g_persist_trace[31] = t;
  }
#endif
  // forward, loss, reverse walk and the norm partials of each sample (no grid barrier: a sample's
  // chain is local to its CTA)
  sample_phase(p, sm);
  grid_sync(p.bar);
  // factors (optimizer.hpp:90-98)
  for (int64_t n = gtid(); n < p.b; n += gstride()) {
    double sq = 0.0;
    for (int pi = 0; pi < p.np; ++pi) sq += __ldcg(p.part + (int64_t)pi * p.b + n);
    const double norm = sqrt(sq);
    const double s = p.c / (norm < p.c ? p.c : norm);
    p.norms[n] = norm;
    p.scale[n] = (float)s;
    if (norm > p.c && p.num_clipped) atomicAdd(reinterpret_cast<unsigned long long*>(p.num_clipped), 1ull);
  }
  grid_sync(p.bar);
  // clipped sum from the record, the reference's order: summed[j] = sum over n ascending of
  // scale[n] * g_n[j] (fp32 multiply, then add)
  for (int64_t j = gtid(); j < p.Ltot; j += gstride()) {
    int pi = 0;
    while (pi + 1 < p.np && j >= p.off[pi + 1]) ++pi;
    const int64_t r = j - p.off[pi];
    const float* g = p.rec[pi] + r;
    const int64_t ne = p.numel[pi];
    float acc = 0.f;
    int64_t n = 0;
    for (; n + 16 <= p.b; n += 16) {  // 16 loads in flight, then the in-order sum
      float v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(g + (n + u) * ne);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, __fmul_rn(__ldcg(p.scale + n + u), v[u]));
    }
    for (; n < p.b; ++n) acc = __fadd_rn(acc, __fmul_rn(__ldcg(p.scale + n), __ldcg(g + n * ne)));
    p.summed[j] = acc;
  }
  grid_sync(p.bar);
  // noise + update (noise.cu's arithmetic), skipped when an error is pending
  if (p.step_ptr && gtid() == 0) *p.step_ptr = step + 1;
  if (error_pending(p.err)) return;
  for (int64_t q = gtid(); 2 * q < p.Ltot; q += gstride()) {
    const int64_t i0 = 2 * q;
    float nz[2] = {0.f, 0.f};
    if (p.injected) {
      nz[0] = p.injected[i0];
      if (i0 + 1 < p.Ltot) nz[1] = p.injected[i0 + 1];
    } else if (p.std_dev != 0.0) {
      double z0, z1;
      normal_pair(p.seed, step, (uint64_t)q, z0, z1);
      nz[0] = (float)(z0 * p.std_dev);
      nz[1] = (float)(z1 * p.std_dev);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int64_t i = i0 + k;
      if (i >= p.Ltot) break;
      const float s = __ldcg(p.summed + i);
      const float noised = (p.injected || p.std_dev != 0.0) ? __fadd_rn(s, nz[k]) : s;
      const float g = __fmul_rn(noised, p.inv_e);
      p.params[i] = __fsub_rn(p.params[i], __fmul_rn(g, p.lr));
      if (p.grad) p.grad[i] = g;
    }
  }
}

}  // namespace ps

#ifdef DPG_PERSIST_TRACE
extern "C" __attribute__((visibility("default"))) void dpg_persist_trace_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, ps::g_persist_trace, sizeof(unsigned long long) * 32);
  int z = 0;
  cudaMemcpyToSymbol(ps::g_persist_ev, &z, sizeof(int));
}
#endif

// host: launch with every CTA co-resident (cooperative launch; the grid barrier needs it)
void launch_persist_step(dpg_ctx* ctx, const ps::Params& p, int smem) {
  ensure_smem_attr(reinterpret_cast<const void*>(ps::persist_step_kernel), smem);
  int per_sm = 0;
  DPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ps::persist_step_kernel, ps::kThreads, smem));
  per_sm = std::max(1, std::min(per_sm, 1));  // one CTA per SM: fewer barrier participants
  void* args[] = {const_cast<ps::Params*>(&p)};
  DPG_CUDA(cudaLaunchCooperativeKernel((const void*)ps::persist_step_kernel, dim3(kNumSMs * per_sm),
                                       dim3(ps::kThreads), args, (size_t)smem, ctx->stream));
  DPG_LAUNCH_CHECK(ctx);
}

}  // namespace dpg
