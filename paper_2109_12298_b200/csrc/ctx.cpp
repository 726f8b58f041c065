// ctx.cpp — dpg_ctx: stream, device error record, workspace, NCCL communicator.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include <vector>

#include "dpg_internal.h"

namespace dpg {

void ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  DPG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{dev, fn}];
  if (bytes <= have) return;
  DPG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

std::string& thread_err() {
  static thread_local std::string s;
  return s;
}

void sync_ctx(dpg_ctx* ctx) {
  DPG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (cudaStream_t s : ctx->extra_streams) DPG_CUDA(cudaStreamSynchronize(s));  // e.g. host read-backs
}

static std::string fmt_value(uint64_t bits) {
  float f;
  uint32_t u = (uint32_t)bits;
  std::memcpy(&f, &u, sizeof f);
  return std::to_string((double)f);
}

void throw_device_error(dpg_ctx* ctx, ErrNamer names, const void* user) {
  sync_ctx(ctx);
  DPG_CUDA(cudaMemcpy(ctx->host_err, ctx->dev_err, sizeof(DeviceErr), cudaMemcpyDeviceToHost));
  const DeviceErr e = *ctx->host_err;
  if (e.key == ERR_NONE) return;
  // clear for the next step
  DeviceErr clear{ERR_NONE, 0};
  *ctx->host_err = clear;
  DPG_CUDA(cudaMemcpy(ctx->dev_err, ctx->host_err, sizeof(DeviceErr), cudaMemcpyHostToDevice));
  const uint64_t stage = e.key >> 56, major = (e.key >> 32) & 0xFFFFFFull, minor = e.key & 0xFFFFFFFFull;
  const std::string who = names ? names(user, stage, major) : std::string();
  switch (stage) {
    case ERR_STAGE_EMBED_INDEX:
      // require_integral_index (layers.hpp:368-376)
      raise(DPG_ERR_PARAMETER, "embedding index " + fmt_value(e.aux) + " out of range" + who +
                                   " (position " + std::to_string(minor) + ")");
    case ERR_STAGE_TARGET:
      raise(DPG_ERR_PARAMETER, "target class " + fmt_value(e.aux) + " out of range" + who +
                                   " (sample " + std::to_string(minor) + ")");
    case ERR_STAGE_NONFINITE:
      // optimizer.hpp:81-82
      raise(DPG_ERR_NUMERIC, "non-finite per-sample gradient in " +
                                 (who.empty() ? "parameter " + std::to_string(major) : who) +
                                 " (sample " + std::to_string(minor) + ")");
    case ERR_STAGE_REMOTE:
      raise(DPG_ERR_NUMERIC, "another rank of the sample-sharded step reported an error; the update "
                             "was skipped on every rank");
    default:
      raise(DPG_ERR_INTERNAL, "unknown device error record");
  }
}

static cudaEvent_t pooled_event(dpg_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  DPG_CUDA(cudaEventCreate(&e));
  return e;
}

ProfScope::ProfScope(dpg_ctx* c, std::string name, double bytes, double flops)
    : ctx(c), on(c->profiling && !c->capturing) {
  if (c->timeline && c->capturing) {  // an event-record node pair inside the captured step
    tl = true;
    rec.name = std::move(name);
    rec.bytes = bytes;
    rec.flops = flops;
    rec.a = pooled_event(ctx);
    rec.b = pooled_event(ctx);
    rec.kernels = ctx->launches;
    rec.seq = (int64_t)ctx->tl_recs.size();
    DPG_CUDA(cudaEventRecordWithFlags(rec.a, ctx->stream, cudaEventRecordExternal));
    return;
  }
  if (!on) return;
  rec.name = std::move(name);
  rec.bytes = bytes;
  rec.flops = flops;
  rec.a = pooled_event(ctx);
  rec.b = pooled_event(ctx);
  rec.kernels = ctx->launches;
  rec.seq = ctx->prof_seq++;
  DPG_CUDA(cudaEventRecord(rec.a, ctx->stream));
}

ProfScope::~ProfScope() {
  if (tl) {
    rec.kernels = ctx->launches - rec.kernels;
    cudaEventRecordWithFlags(rec.b, ctx->stream, cudaEventRecordExternal);
    ctx->tl_recs.push_back(rec);
    return;
  }
  if (!on) return;
  rec.kernels = ctx->launches - rec.kernels;
  cudaEventRecord(rec.b, ctx->stream);
  ctx->prof_pending.push_back(rec);
}

}  // namespace dpg

void* dpg_ctx::workspace(size_t bytes) {
  if (bytes <= ws_bytes) return ws;
  if (capturing) dpg::raise(DPG_ERR_INTERNAL, "workspace growth during graph capture");
  DPG_CUDA(cudaStreamSynchronize(stream));
  if (ws) DPG_CUDA(cudaFree(ws));
  ws = nullptr;
  ws_bytes = 0;
  const size_t want = bytes < (1u << 20) ? (1u << 20) : bytes;
  DPG_CUDA(cudaMalloc(&ws, want));
  ws_bytes = want;
  return ws;
}

const int32_t* dpg_ctx::identity_rows(int n) {
  if (n <= iota_n) return iota;
  if (capturing) dpg::raise(DPG_ERR_INTERNAL, "identity-row table growth during graph capture");
  const int cap = n < 1024 ? 1024 : n;
  std::vector<int32_t> h(cap);
  for (int i = 0; i < cap; ++i) h[i] = i;
  DPG_CUDA(cudaStreamSynchronize(stream));
  if (iota) DPG_CUDA(cudaFree(iota));
  iota = nullptr;
  iota_n = 0;
  DPG_CUDA(cudaMalloc(&iota, sizeof(int32_t) * cap));
  DPG_CUDA(cudaMemcpy(iota, h.data(), sizeof(int32_t) * cap, cudaMemcpyHostToDevice));
  iota_n = cap;
  return iota;
}

bool dpg_ctx::can_fork() {
  if (side) return true;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &st) != cudaSuccess) return false;
  return st == cudaStreamCaptureStatusNone && !capturing;
}

void dpg_ctx::fork_side() {
  if (!side) {
    DPG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    DPG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    DPG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  }
  main_saved = stream;
  DPG_CUDA(cudaEventRecord(ev_fork, stream));
  DPG_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
  stream = side;
}

void dpg_ctx::end_side() {
  DPG_CUDA(cudaEventRecord(ev_join, side));
  stream = main_saved;
}

void dpg_ctx::join_side() { DPG_CUDA(cudaStreamWaitEvent(stream, ev_join, 0)); }

using dpg::guard;

extern "C" {

int dpg_abi_version(void) { return DPG_ABI_VERSION; }

dpg_status dpg_ctx_create(int device, void* stream, dpg_ctx** out) {
  if (!out) return DPG_ERR_PARAMETER;
  *out = nullptr;
  dpg_ctx* ctx = new dpg_ctx();
  const dpg_status st = guard(nullptr, [&] {
    int count = 0;
    DPG_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      dpg::raise(DPG_ERR_PARAMETER, "device " + std::to_string(device) + " out of range");
    ctx->device = device;
    DPG_CUDA(cudaSetDevice(device));
    int major = 0, minor = 0;
    DPG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    DPG_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
      dpg::raise(DPG_ERR_CUDA, "libdpg is built for sm_100a (B200); device has compute capability " +
                                   std::to_string(major) + "." + std::to_string(minor));
    if (stream) {
      ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
      DPG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
    DPG_CUDA(cudaMalloc(&ctx->dev_err, sizeof(dpg::DeviceErr)));
    DPG_CUDA(cudaMalloc(&ctx->clip_sync, 2 * sizeof(unsigned long long)));
    DPG_CUDA(cudaMemset(ctx->clip_sync, 0, 2 * sizeof(unsigned long long)));
    DPG_CUDA(cudaMallocHost(&ctx->host_err, sizeof(dpg::DeviceErr)));
    dpg::DeviceErr clear{dpg::ERR_NONE, 0};
    *ctx->host_err = clear;
    DPG_CUDA(cudaMemcpy(ctx->dev_err, ctx->host_err, sizeof(clear), cudaMemcpyHostToDevice));
  });
  if (st != DPG_OK) {
    delete ctx;
    return st;
  }
  *out = ctx;
  return DPG_OK;
}

void dpg_ctx_destroy(dpg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->iota) cudaFree(ctx->iota);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
  }
  if (ctx->dev_err) cudaFree(ctx->dev_err);
  if (ctx->clip_sync) cudaFree(ctx->clip_sync);
  if (ctx->host_err) cudaFreeHost(ctx->host_err);
  for (auto& r : ctx->prof_pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

void* dpg_ctx_stream(const dpg_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

const char* dpg_last_error(const dpg_ctx* ctx) {
  return ctx ? ctx->err.c_str() : dpg::thread_err().c_str();
}

dpg_status dpg_ctx_sync(dpg_ctx* ctx) {
  if (!ctx) return DPG_ERR_PARAMETER;
  return guard(ctx, [&] { dpg::throw_device_error(ctx, nullptr, nullptr); });
}

int64_t dpg_ctx_kernel_launches(const dpg_ctx* ctx) { return ctx ? ctx->launches : 0; }

dpg_status dpg_ctx_set_profiling(dpg_ctx* ctx, int on) {
  if (!ctx) return DPG_ERR_PARAMETER;
  return guard(ctx, [&] {
    ctx->profiling = on != 0;
    if (on) {
      ctx->prof_agg.clear();
      ctx->prof_seq = 0;
    }
  });
}

dpg_status dpg_ctx_set_timeline(dpg_ctx* ctx, int on) {
  if (!ctx) return DPG_ERR_PARAMETER;
  return guard(ctx, [&] {
    if (ctx->capturing) dpg::raise(DPG_ERR_LIFECYCLE, "set_timeline during a graph capture");
    ctx->timeline = on != 0;
    for (auto& r : ctx->tl_recs) {
      ctx->event_pool.push_back(r.a);
      ctx->event_pool.push_back(r.b);
    }
    ctx->tl_recs.clear();
    if (on && !ctx->tl_start) DPG_CUDA(cudaEventCreate(&ctx->tl_start));
  });
}

const char* dpg_ctx_timeline_read(dpg_ctx* ctx) {
  if (!ctx) return "";
  const dpg_status st = guard(ctx, [&] {
    DPG_CUDA(cudaDeviceSynchronize());
    std::string out;
    char line[512];
    for (auto& r : ctx->tl_recs) {
      float t0 = 0.f, dt = 0.f;
      DPG_CUDA(cudaEventElapsedTime(&t0, ctx->tl_start, r.a));
      DPG_CUDA(cudaEventElapsedTime(&dt, r.a, r.b));
      std::snprintf(line, sizeof line, "%s %.6f %.6f %lld\n", r.name.c_str(), t0, dt, (long long)r.kernels);
      out += line;
    }
    ctx->prof_text = out;
  });
  if (st != DPG_OK) return "";
  return ctx->prof_text.c_str();
}

const char* dpg_ctx_profile_read(dpg_ctx* ctx) {
  if (!ctx) return "";
  const dpg_status st = guard(ctx, [&] {
    DPG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& r : ctx->prof_pending) {
      float ms = 0.f;
      DPG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      auto& a = ctx->prof_agg[r.name];
      a.ms += ms;
      a.bytes += r.bytes;
      a.flops += r.flops;
      a.count += 1;
      a.kernels += r.kernels;
      if (a.first_seq < 0) a.first_seq = r.seq;
      ctx->event_pool.push_back(r.a);
      ctx->event_pool.push_back(r.b);
    }
    ctx->prof_pending.clear();
    std::string out;
    char line[512];
    for (auto& [name, a] : ctx->prof_agg) {
      std::snprintf(line, sizeof line, "%s %.6f %lld %.1f %.1f %lld %lld\n", name.c_str(), a.ms,
                    (long long)a.count, a.bytes, a.flops, (long long)a.kernels, (long long)a.first_seq);
      out += line;
    }
    ctx->prof_text = out;
  });
  if (st != DPG_OK) return "";
  return ctx->prof_text.c_str();
}

dpg_status dpg_nccl_unique_id(unsigned char id[128]) {
  return guard(nullptr, [&] {
    ncclUniqueId uid;
    DPG_NCCL(ncclGetUniqueId(&uid));
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, uid.internal, 128);
  });
}

dpg_status dpg_ctx_init_comm(dpg_ctx* ctx, int nranks, int rank, const unsigned char id[128]) {
  if (!ctx) return DPG_ERR_PARAMETER;
  return guard(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) dpg::raise(DPG_ERR_PARAMETER, "bad rank / nranks");
    DPG_CUDA(cudaSetDevice(ctx->device));
    if (ctx->comm) {
      DPG_NCCL(ncclCommDestroy(ctx->comm));
      ctx->comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    ++ctx->comm_gen;  // (also when the init below fails: graphs holding the old comm are stale)
    DPG_NCCL(ncclCommInitRank(&ctx->comm, nranks, uid, rank));
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

dpg_status dpg_allreduce_sum(dpg_ctx* ctx, float* buf, int64_t n) {
  if (!ctx) return DPG_ERR_PARAMETER;
  return guard(ctx, [&] {
    if (!ctx->comm) dpg::raise(DPG_ERR_LIFECYCLE, "allreduce without a communicator (dpg_ctx_init_comm)");
    DPG_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, ctx->comm, ctx->stream));
  });
}

}  // extern "C"

