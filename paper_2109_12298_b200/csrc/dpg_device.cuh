// dpg_device.cuh — device-side helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

#include "dpg_internal.h"

namespace dpg {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

__device__ __forceinline__ float relu_if(float v, int relu) { return (relu && !(v > 0.f)) ? 0.f : v; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree): every thread passes its value, thread 0 gets the total.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* smem /* >= NT/32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < NT / 32 ? smem[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// Zero word that out-of-range gathers load from: operand loads are unconditional (the address is
// selected, not the load), so a thread's gathers are all in flight at once and nothing consumes
// a loaded value before it is needed.
static __device__ __align__(16) const float g_zero4[4] = {0.f, 0.f, 0.f, 0.f};

// Load *p when ok, else the zero word. The address is selected with selp (both candidates are
// computed unconditionally), so the compiler cannot turn the gather into a branch per element.
__device__ __forceinline__ float ldg_or_zero(const float* p, bool ok) {
  const float* q;
  asm("{\n\t.reg .pred sel;\n\tsetp.ne.b32 sel, %3, 0;\n\tselp.b64 %0, %1, %2, sel;\n\t}"
      : "=l"(q)
      : "l"(p), "l"(g_zero4), "r"((int)ok));
  return __ldg(q);
}
__device__ __forceinline__ float4 ldg4_or_zero(const float* p, bool ok) {
  const float* q;
  asm("{\n\t.reg .pred sel;\n\tsetp.ne.b32 sel, %3, 0;\n\tselp.b64 %0, %1, %2, sel;\n\t}"
      : "=l"(q)
      : "l"(p), "l"(g_zero4), "r"((int)ok));
  return __ldg(reinterpret_cast<const float4*>(q));
}

// Record (key, aux) if key precedes the recorded key. Key and aux change together under a lock
// word, so the aux always belongs to the recorded key (errors are rare: the lock is off the fast
// path, which is one relaxed read).
__device__ __forceinline__ void report_error(DeviceErr* err, uint64_t key, uint64_t aux) {
  if (key >= *(volatile unsigned long long*)&err->key) return;
  while (atomicCAS(&err->lock, 0u, 1u) != 0u) __nanosleep(32);
  __threadfence();
  if (key < *(volatile unsigned long long*)&err->key) {
    *(volatile unsigned long long*)&err->aux = aux;
    __threadfence();
    *(volatile unsigned long long*)&err->key = key;
  }
  __threadfence();
  atomicExch(&err->lock, 0u);
}

__device__ __forceinline__ bool error_pending(const DeviceErr* err) {
  return *(volatile const unsigned long long*)&err->key != ERR_NONE;
}

// streaming store for write-once outputs (per-sample gradients)
__device__ __forceinline__ void st_stream4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Programmatic dependent launch: every kernel is launched with programmatic stream
// serialization (launch_pdl), so it may start — and run its prologue — while the previous kernel
// on the stream drains; pdl_wait() (griddepcontrol.wait) blocks until that kernel has completed
// and its memory is visible. Every kernel calls it before touching data another kernel wrote.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the next kernel on the stream launch before this one finishes (its own pdl_wait still
// waits for this grid's completion and memory)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch with programmatic stream serialization (see pdl_wait); DPG_PDL=0 launches plainly.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DPG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);  // errors: DPG_LAUNCH_CHECK
}

}  // namespace dpg
