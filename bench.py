#!/usr/bin/env python
"""bench.py — DP-SGD step throughput of the B200 path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

One "step" is one full DP-SGD step (forward, per-sample gradients with fused norms, clip factors,
clipped sum, [NCCL all-reduce], noise + SGD update) over one synthetic batch, replayed from a
CUDA graph. N=1 runs BASELINE configs[2] (CIFAR-10 4-layer CNN, batch 512); N>1 (torchrun, one
rank per GPU) shards by sample with 512 samples per rank (weak scaling; N=8 is configs[4]'s
global batch 4096) and one all-reduce of the clipped sum per step.

Reported (rank 0 prints ONE JSON line):
  value        samples/s over all ranks, inputs resident in HBM, device time (CUDA events on the
               launching stream), L2 flushed (256 MiB write) before every timed step, max over ranks
  e2e          the same metric through dpg_train_step_host_async with pinned HOST buffers: H2D of
               the batch and D2H of the per-sample loss inside the timed region every step (the
               copies of step k + 1 overlap the kernels of step k)
  roofline     dominant stage of an eager profiled pass: algorithmic bytes / its CUDA-event
               duration vs the measured HBM peak; plus the whole-step fraction
  cpu_baseline the reference compiled from its own sources (oracle/_ref, -O3), sample-sharded
               over all host cores, timed on this box (rank 0, N=1 only)
  --impl reference: the reference CPU path alone (rank 0), same metric / config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DP-SGD step samples/sec (CIFAR-10 CNN, B=512)"
METRICS = {"cifar_b512": METRIC,
           "mnist_b64": "DP-SGD step samples/sec (MNIST CNN, B=64)",
           "embed_b512": "DP-SGD step samples/sec (Embedding 10000x128 + Linear, T=256, B=512)",
           "cifar_b4096": "DP-SGD step samples/sec (CIFAR-10 CNN, B=4096)"}
HBM_FALLBACK = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cifar_b512")
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--max-grad-norm", type=float, default=1.0)
    ap.add_argument("--no-materialise", action="store_true",
                    help="norms without storing the GradSampleRecord (not the headline)")
    ap.add_argument("--csum-from-record", action="store_true",
                    help="clipped sums as the reference's pass 2 over the stored record (not the headline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["p2p", "nccl"],
                    help="N > 1: one NCCL all-reduce of the clipped sum (default), or the exchange "
                         "over peer memory inside the update kernel (dpg_optimizer_set_peers)")
    ap.add_argument("--no-strong", action="store_true",
                    help="skip the strong-scaling cfg5 line (global batch 4096 split over the ranks)")
    ap.add_argument("--profile-steps", type=int, default=5)
    return ap.parse_args()


def dist_env():
    # DPG_BENCH_DEVICE pins every rank to one device: a protocol check of the N > 1 path on a
    # one-GPU box (the peer exchange works between processes sharing a GPU); not a measurement
    local = int(os.environ.get("DPG_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), local


def spawn_ranks(nranks: int) -> int:
    """`bench.py --gpus N` started without torchrun: re-launch this command as N ranks under
    torch.distributed.run on 127.0.0.1 (the driver's own form); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_for(workload_name: str, global_batch: int, per_rank: int, world: int, detail: dict) -> dict:
    """The `config` object, with the same keys in both arms (detail: arm-specific settings)."""
    return {"workload": workload_name, "global_batch": global_batch, "per_rank_batch": per_rank,
            "parallelism": f"dp{world} (sample shards)" if world > 1 else "dp1 (one GPU)", "detail": detail}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK, "fallback"


# ------------------------------------------------------------------------------ synthetic data
def synth(workload, b, seed_params=1, seed_data=2):
    """Random-init weights of the workload's architecture (U(+-1/sqrt(fan_in)), N(0,1) tables,
    as build_model does) and a synthetic batch; numpy only, no oracle involved."""
    import numpy as np
    from paper_2109_12298_b200.configs import CONV2D, EMBEDDING, LINEAR, param_count
    rng = np.random.default_rng(seed_params)
    ps = []
    for l in workload.layers:
        if l.kind == LINEAR:
            k = 1 / np.sqrt(l.in_features)
            ps.append(rng.uniform(-k, k, l.out_features * l.in_features))
            if l.has_bias:
                ps.append(rng.uniform(-k, k, l.out_features))
        elif l.kind == CONV2D:
            k = 1 / np.sqrt(l.in_channels * l.kernel_h * l.kernel_w)
            ps.append(rng.uniform(-k, k, l.out_channels * l.in_channels * l.kernel_h * l.kernel_w))
            if l.has_bias:
                ps.append(rng.uniform(-k, k, l.out_channels))
        elif l.kind == EMBEDDING:
            ps.append(rng.standard_normal(l.vocab_size * l.embedding_dim))
    params = np.concatenate(ps).astype(np.float32)
    assert params.size == param_count(workload.layers)
    drng = np.random.default_rng(seed_data)
    if workload.tokens:
        x = drng.integers(0, workload.tokens, size=(b,) + workload.in_shape).astype(np.float32)
    else:
        x = drng.standard_normal((b,) + workload.in_shape).astype(np.float32)
    y = drng.integers(0, workload.classes, size=b).astype(np.float32)
    return params, x, y


def step_bytes(workload, b, materialise=True):
    """B_hot = 4[sum(|X_l| + |Y_l|) + b L + 4 L];
    B_full = B_hot + forward sum 4(|X_l| + |Y_l|) + backward sum_{l>0} 4(|Y_l| + 2|X_l|)."""
    from paper_2109_12298_b200.configs import CONV2D, EMBEDDING, FLATTEN, LINEAR, param_count
    L = param_count(workload.layers)
    shape = list(workload.in_shape)
    xs, ys = [], []
    for l in workload.layers:
        n_in = 1
        for e in shape:
            n_in *= e
        if l.kind == LINEAR:
            shape[-1] = l.out_features
        elif l.kind == CONV2D:
            oh = (shape[1] + 2 * l.padding - l.kernel_h) // l.stride + 1
            ow = (shape[2] + 2 * l.padding - l.kernel_w) // l.stride + 1
            shape = [l.out_channels, oh, ow]
        elif l.kind == EMBEDDING:
            shape = [shape[0], l.embedding_dim]
        elif l.kind == FLATTEN:
            shape = [n_in]
        else:
            continue
        if l.kind in (LINEAR, CONV2D, EMBEDDING):
            n_out = 1
            for e in shape:
                n_out *= e
            xs.append(b * n_in)
            ys.append(b * n_out)
    hot = 4 * (sum(xs) + sum(ys) + (b * L if materialise else 0) + 4 * L)
    fwd = 4 * (sum(xs) + sum(ys))
    bwd = 4 * sum(ys[i] + 2 * xs[i] for i in range(1, len(xs)))
    return hot, hot + fwd + bwd


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled every ~2 ms from a
    thread (nvidia-smi -lms buffers its pipe and loses a short window's samples)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        self.index = int(ids[index]) if index < len(ids) and ids[index].isdigit() else index
        self.samples = []
        self.stop_ev = threading.Event()
        self.err = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            get = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.get_reasons = get
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv, h = self.nv, self.h
        while True:
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), self.get_reasons(h)))
            except Exception:  # noqa: BLE001
                pass
            if self.stop_ev.is_set():  # the sample taken after stop() closes the window
                break
            time.sleep(0.002)

    def stop(self):
        if self.err:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err], "samples": 0}
        self.stop_ev.set()
        self.t.join(timeout=2)
        reasons = set()
        for _, r in self.samples:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        sm = [c for c, _ in self.samples]
        loaded = [c for c in sm if c > 0.5 * self.smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": self.smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------ reference arm
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_sample_step(workload, b_sample, nthreads, fast=True):
    """One DP-SGD step of the reference over b_sample samples of the workload; returns seconds
    and the kind used. oracle/_ref (the reference built from its sources) when present."""
    import numpy as np
    import oracle
    params, x, y = synth(workload, b_sample)
    if oracle.reference_available(fast=fast):
        ref = oracle.reference(fast=fast)
        t0 = time.perf_counter()
        ref.dpsgd_step_threads(workload.layers, workload.in_shape, params, x, y, 1.0, 1.0, 0.1,
                               float(b_sample), 3, nthreads)
        return time.perf_counter() - t0, "reference", nthreads
    r = oracle.restatement()
    t0 = time.perf_counter()
    r.dpsgd_step(workload.layers, workload.in_shape, params, x, y, 1.0, 1.0, 0.1, float(b_sample),
                 want_record=False)
    return time.perf_counter() - t0, "port", 1


def pick_sample(workload, nthreads, budget_s):
    """Largest sample (multiple of nthreads, <= workload batch) whose step fits budget_s."""
    b = max(nthreads, 8)
    t, kind, cores = reference_sample_step(workload, b, nthreads)
    per_sample = t / b
    want = int(budget_s / max(per_sample, 1e-9))
    want = max(b, min(workload.batch, want))
    want -= want % max(1, min(nthreads, want))
    return max(b, want), kind, cores


def cpu_baseline(workload, budget_s=15.0, single_thread=True):
    """The reference on this box's host cores: sample-sharded over all threads (the headline
    baseline) and, as BASELINE.md §3.1 item 5 asks, the reference as-is on one thread."""
    nthreads = cpu_threads()
    b, kind, cores = pick_sample(workload, nthreads, budget_s / 3)
    times = []
    t_end = time.perf_counter() + budget_s
    while True:
        t, kind, cores = reference_sample_step(workload, b, nthreads)
        times.append(t)
        if time.perf_counter() > t_end or len(times) >= 10:
            break
    med = statistics.median(times)
    out = {"value": b / med, "unit": "samples/s", "cores": cores, "kind": kind,
           "sample": f"{workload.name}: full DP-SGD step of the reference over {b} samples, "
                     f"median of {len(times)} steps, {'-O3 -march=x86-64-v3 ' if kind == 'reference' else ''}"
                     f"{cores} host threads (sample-sharded, virtual-step semantics)"}
    if single_thread and cores > 1:
        b1, kind1, _ = pick_sample(workload, 1, 2.0)
        t1 = [reference_sample_step(workload, b1, 1)[0] for _ in range(3)]
        out["single_thread"] = {"value": b1 / statistics.median(t1), "unit": "samples/s", "cores": 1,
                                "kind": kind1, "sample": f"{b1} samples per step, median of 3 steps, one thread"}
    return out


def linear_t64_config(args):
    """The cfg2 config dict, identical in both arms."""
    from paper_2109_12298_b200.configs import LINEAR_T64 as C
    return {"workload": "linear_t64", "batch": C["b"], "seq_len": C["t"], "in": C["d"],
            "out": C["r"], "sigma": args.sigma, "max_grad_norm": args.max_grad_norm,
            "l2": "no flush: the 268 MB per-sample gradient exceeds L2 every step"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.workload == "linear_t64":
        cb = cpu_baseline_linear_t64(budget_s=60.0)
        line = {"metric": LINEAR_T64_METRIC, "value": cb["value"], "unit": "samples/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
                "config": linear_t64_config(args), "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    from paper_2109_12298_b200.configs import WORKLOADS
    w = WORKLOADS[args.workload]
    nthreads = cpu_threads()
    # size each step so warmup + steps finish in about two minutes
    b, kind, cores = pick_sample(w, nthreads, 120.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        reference_sample_step(w, b, nthreads)
    total = 0.0
    for _ in range(args.steps):
        t, kind, cores = reference_sample_step(w, b, nthreads)
        total += t
    value = b * args.steps / total
    line = {
        "metric": METRICS.get(w.name, METRIC), "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": config_for(w.name, w.batch * args.gpus, w.batch, args.gpus,
                             {"arm": "reference CPU path", "per_step_sample": b}),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind,
                         "sample": f"{b} samples of {w.name} per step, {cores} host threads"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ cfg2 harness
LINEAR_T64_METRIC = "DP-SGD per-layer step samples/sec (Linear 512->512, T=64, B=256)"


def tf32_peak_tflops():
    """Dense TF32 tensor throughput measured here (torch.matmul 8192^3, allow_tf32, best of 5)."""
    import torch
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    best = 1e9
    try:
        for _ in range(2):
            a @ b
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def run_linear_t64(args, rank, world):
    """BASELINE configs[1]: per_sample_rule_linear on A, B [256, 64, 512] (tcgen05 3xTF32, fused
    norms) + bias rule -> clip factors -> clipped sum (s . B)^T A -> noise + SGD update, through
    the operator ABI (dpg_grad_sample_linear, dpg_clip_factors, dpg_clipped_sum_linear,
    dpg_noise_update) on device-resident buffers."""
    import ctypes
    import torch
    from paper_2109_12298_b200 import dpg
    from paper_2109_12298_b200.configs import LINEAR_T64 as C
    torch.cuda.set_device(0)
    ctx = dpg.Context(0)
    lib = dpg.lib()
    b, t, d, r = C["b"], C["t"], C["d"], C["r"]
    L = r * d + r
    g = torch.Generator(device="cpu").manual_seed(2)
    A = torch.randn(b, t, d, generator=g).cuda()
    B = torch.randn(b, t, r, generator=g).cuda()
    gw = torch.empty(b, r, d, device="cuda")
    gb = torch.empty(b, r, device="cuda")
    sq = torch.empty(2, b, dtype=torch.float64, device="cuda")
    norms = torch.empty(b, dtype=torch.float64, device="cuda")
    scale = torch.empty(b, device="cuda")
    nclip = torch.zeros(1, dtype=torch.int64, device="cuda")
    summed = torch.empty(L, device="cuda")
    params = (torch.rand(L, generator=g) - 0.5).cuda() / d ** 0.5
    grad = torch.empty(L, device="cuda")
    P = dpg._p
    step_no = [0]

    def stages():
        return [
            ("gs.linear+bias", lambda: dpg._check(lib.dpg_grad_sample_linear(
                ctx.h, P(A), P(B), b, t, d, r, P(gw), P(gb), P(sq[0]), P(sq[1])), ctx.h),
             4.0 * (b * t * (d + r) + b * r * d + b * r), 2.0 * b * t * d * r),
            ("clip_factors", lambda: dpg._check(lib.dpg_clip_factors(
                ctx.h, P(sq), 2, b, args.max_grad_norm, P(norms), P(scale), P(nclip)), ctx.h),
             8.0 * 2 * b + 12.0 * b, 0.0),
            ("csum.linear+bias", lambda: dpg._check(lib.dpg_clipped_sum_linear(
                ctx.h, P(A), P(B), P(scale), b, t, d, r, P(summed), P(summed[r * d:]), 0), ctx.h),
             4.0 * (b * t * (d + r) + 2 * L), 2.0 * b * t * d * r),
            ("noise_update", lambda: dpg._check(lib.dpg_noise_update(
                ctx.h, P(params), P(summed), P(grad), L, args.sigma, args.max_grad_norm, float(b), 0.1,
                3, step_no[0], None), ctx.h), 16.0 * L, 0.0),
        ]

    st = stages()

    def step():
        for _, f, _, _ in st:
            f()
        step_no[0] += 1

    stream = ctx.stream
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    launches0 = ctx.kernel_launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    gpu_launches = ctx.kernel_launches - launches0
    ctx.sync()
    total_ms = sum(a.elapsed_time(c) for a, c in evs)
    value = b * args.steps / (total_ms / 1000.0)
    # per-stage device time (events around each stage; G = 268 MB > L2, so no flush is needed)
    per = {name: 0.0 for name, _, _, _ in st}
    reps = 10
    for _ in range(reps):
        for name, f, _, _ in st:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            f()
            e1.record(stream)
            torch.cuda.synchronize()
            per[name] += e0.elapsed_time(e1) / reps
    hbm, peak_src = peaks()
    tf32 = tf32_peak_tflops()
    name, _, by, fl = st[0]
    ms = per[name]
    achieved_gbs = by / (ms * 1e6)
    achieved_tf = fl / (ms * 1e9)
    # DRAM bytes of the dominant stage from a committed ncu capture (tools/lin_traffic.py)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic_linear_t64.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        if name in tj:
            traffic = tj[name]["traffic"]
            traffic_src = (f"committed capture {os.path.relpath(tpath, ROOT)} ({tj.get('_source', 'ncu')}); "
                           "not measured in this run")
    # end to end: pinned host A, B -> device, step, norms back
    Ah, Bh = A.cpu().pin_memory(), B.cpu().pin_memory()
    nh = torch.empty(b, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        A.copy_(Ah, non_blocking=True)
        B.copy_(Bh, non_blocking=True)
        step()
        nh.copy_(norms, non_blocking=True)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    line = {
        "metric": LINEAR_T64_METRIC, "value": value, "unit": "samples/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": linear_t64_config(args),
        "roofline": {"bound": "hbm", "kernel": name, "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": achieved_gbs / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                     "algorithmic_bytes_per_launch": by, "launch_ms": ms,
                     "tensor": {"achieved_tflops": achieved_tf, "tf32_peak_tflops_measured": tf32,
                                "peak_3xtf32_tflops": tf32 / 3.0, "frac_3xtf32": achieved_tf / (tf32 / 3.0)},
                     # every contraction stage against both rooflines (the clipped sum is the
                     # tensor-bound one: 2 b T d r flops over only 4 b T (d + r) bytes)
                     "stages": {sn: {"ms": per[sn], "hbm_frac": sb / (per[sn] * 1e6) / hbm,
                                     "tflops": sf / (per[sn] * 1e9),
                                     "frac_3xtf32": sf / (per[sn] * 1e9) / (tf32 / 3.0)}
                                for sn, _, sb, sf in st if sf > 0},
                     "stages_ms": per},
        "e2e": {"value": b * args.steps / e2e_s, "unit": "samples/s",
                "h2d_bytes_per_step": int(A.numel() + B.numel()) * 4, "d2h_bytes_per_step": b * 8},
        "gpu_launches": gpu_launches, "clocks": clk,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_linear_t64()
    print(json.dumps(line), flush=True)


def cpu_baseline_linear_t64(budget_s=15.0):
    """The reference's per_sample_rule_linear + clip_and_sum on sample shards (one host thread per
    shard, as the virtual-step thread pool does), then the shard sums added and add_noise, on a
    bounded sample of the cfg2 batch (oracle/_ref built -O3 from the reference's sources)."""
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np
    import oracle
    from paper_2109_12298_b200.configs import LINEAR_T64 as C
    if not oracle.reference_available(fast=True):
        return None
    ref = oracle.reference(fast=True)
    nthreads = cpu_threads()
    b = 2 * nthreads
    rng = np.random.default_rng(2)
    A = rng.standard_normal((b, C["t"], C["d"])).astype(np.float32)
    B = rng.standard_normal((b, C["t"], C["r"])).astype(np.float32)
    shards = np.array_split(np.arange(b), nthreads)

    def shard(ix):
        gw, gb = ref.rule_linear(np.ascontiguousarray(A[ix]), np.ascontiguousarray(B[ix]))
        return ref.clip_and_sum([gw, gb], 1.0)[0]

    times = []
    t_end = time.perf_counter() + budget_s
    with ThreadPoolExecutor(nthreads) as ex:
        while True:
            t0 = time.perf_counter()
            parts = list(ex.map(shard, shards))
            summed = np.concatenate([sum(p[k] for p in parts) for k in range(2)])
            ref.add_noise(summed, 1.0, 1.0, 3)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() > t_end or len(times) >= 5:
                break
    med = statistics.median(times)
    return {"value": b / med, "unit": "samples/s", "cores": nthreads, "kind": "reference",
            "sample": f"linear_t64: {b} samples per step (rule + clip_and_sum per {len(shards)} "
                      f"thread shards, add_noise), median of {len(times)}, -O3 -march=x86-64-v3"}


# ------------------------------------------------------------------------------ Poisson batches
def run_poisson(args):
    """Poisson sampling on the host (data.cpp:31-37: each of N examples joins a
    batch with probability q = E / N), so every step has a different physical batch size; the
    device step replays from the bounded graph cache (updated in place on a miss). E = 512 of a
    CIFAR-10-sized dataset (N = 50000); samples/s = sum of realised batch sizes / device time."""
    import numpy as np
    import torch
    from paper_2109_12298_b200 import dpg
    from paper_2109_12298_b200.configs import WORKLOADS
    w = WORKLOADS["cifar_b512"]
    N, E = 50000, 512
    q = E / N
    rng = np.random.default_rng(7)
    sizes = [int(v) for v in rng.binomial(N, q, size=args.warmup + args.steps)]
    bmax = max(sizes)
    params, _, _ = synth(w, bmax)
    _, x, y = synth(w, bmax)
    ctx = dpg.Context(0)
    model = dpg.Model(ctx, w.layers, w.in_shape, max_batch=bmax)
    model.load_params(params)
    opt = dpg.DpOptimizer(model, noise_multiplier=args.sigma, max_grad_norm=args.max_grad_norm,
                          learning_rate=0.1, expected_batch_size=float(E), noise_seed=3)
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    loss = torch.zeros(bmax, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for b in sizes[:args.warmup]:
        opt.train_step(xt[:b], yt[:b], loss[:b])
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.kernel_launches
    for i, b in enumerate(sizes[args.warmup:]):
        flush.zero_()
        evs[i][0].record(stream)
        opt.train_step(xt[:b], yt[:b], loss[:b])
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ctx.sync()
    total_ms = sum(a.elapsed_time(c) for a, c in evs)
    timed = sizes[args.warmup:]
    line = {
        "metric": "DP-SGD step samples/sec (CIFAR-10 CNN, Poisson sampling, E=512)",
        "value": sum(timed) / (total_ms / 1000.0), "unit": "samples/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "cifar_poisson", "dataset": N, "expected_batch": E, "q": q,
                   "batch_min": min(timed), "batch_max": max(timed), "distinct_batches": len(set(timed)),
                   "graph_cache": "8 executables, LRU, updated in place on a miss",
                   "l2": "256 MiB flush before every timed step (outside the step's events)"},
        "gpu_launches": ctx.kernel_launches - launches0, "clocks": clk,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines name the N ranks
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo")
    if args.workload == "cifar_poisson" and args.impl == "ours":
        if rank == 0:
            run_poisson(args)
        return
    if args.workload == "linear_t64" and args.impl == "ours":
        if rank == 0:
            run_linear_t64(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        return

    import numpy as np
    import torch
    from paper_2109_12298_b200 import dpg
    from paper_2109_12298_b200.configs import WORKLOADS

    ndev = torch.cuda.device_count()
    shared = world > ndev  # more ranks than GPUs (a 1-GPU box): ranks share devices, protocol check only
    if shared:
        local = local % ndev
    torch.cuda.set_device(local)
    ctx = dpg.Context(local)

    w = WORKLOADS[args.workload]
    b = w.batch
    gb = b * world
    params, _, _ = synth(w, b)
    _, x, y = synth(w, b, seed_data=2 + rank)
    model = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
    model.load_params(params)
    materialise = not args.no_materialise
    opt = dpg.DpOptimizer(model, noise_multiplier=args.sigma, max_grad_norm=args.max_grad_norm,
                          learning_rate=0.1, expected_batch_size=float(gb), noise_seed=3,
                          materialise_grad_sample=materialise,
                          clipped_sum_from_record=args.csum_from_record and materialise)
    exchange = args.exchange if world > 1 else None
    if shared and exchange == "nccl":
        exchange = "p2p"  # NCCL refuses two ranks on one device; CUDA IPC within a device works

    def setup_exchange(o, exchange):
        """Wire optimizer o into the chosen exchange; returns the exchange actually used."""
        if exchange == "p2p":
            handles = [None] * world
            torch.distributed.all_gather_object(handles, o.peer_handle())
            err = ""
            try:
                o.set_peers(rank, handles)
            except dpg.DpgError as e:  # e.g. no peer access between these GPUs
                err = str(e)
            errs = [None] * world
            torch.distributed.all_gather_object(errs, err)
            if any(errs):  # every rank must take the same path
                if not err:
                    o.set_peers(rank, [handles[rank]])
                if rank == 0:
                    print(f"peer exchange unavailable ({next(e for e in errs if e)}); using NCCL", file=sys.stderr)
                exchange = "nccl"
        if exchange == "nccl" and not comm_ready[0]:
            obj = [dpg.Context.nccl_unique_id() if rank == 0 else None]
            torch.distributed.broadcast_object_list(obj, src=0)
            ctx.init_comm(world, rank, obj[0])
            comm_ready[0] = True
        return exchange

    comm_ready = [False]
    exchange = setup_exchange(opt, exchange)
    xt = torch.from_numpy(x).cuda()
    yt = torch.from_numpy(y).cuda()
    loss = torch.zeros(b, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- warmup (graph capture happens on the first step) ----
    for _ in range(max(3, args.warmup)):
        opt.train_step(xt, yt, loss)
    ctx.sync()
    # bring SM clocks up before the timed region; rank 0's clock decides when to stop, so every
    # rank runs the same number of steps (each step's exchange pairs across ranks)
    t_soak = time.perf_counter() + 0.5
    while True:
        for _ in range(10):
            opt.train_step(xt, yt, loss)
        torch.cuda.synchronize()
        done = torch.tensor([int(time.perf_counter() >= t_soak)])
        if world > 1:
            torch.distributed.broadcast(done, src=0)
        if done.item():
            break
    barrier()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step CUDA events, L2 flushed before each step ----
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.kernel_launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(stream)
        opt.train_step(xt, yt, loss)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    gpu_launches = ctx.kernel_launches - launches0
    ctx.sync()  # surfaces any device-side error
    step_ms = [a.elapsed_time(c) for a, c in evs]
    total_ms = max_over_ranks(sum(step_ms))
    value = gb * args.steps / (total_ms / 1000.0)

    # ---- end to end: pinned host buffers through dpg_train_step_host_async (per step: H2D of the
    # batch, the step, D2H of the per-sample loss; copies pipelined against the previous step) ----
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.from_numpy(y).pin_memory()
    lh = torch.zeros(b).pin_memory()
    for _ in range(3):
        opt.train_step_host_async(xh, yh, lh)
    ctx.sync()
    barrier()
    # wall clock over >= 2000 steps (~1 s): a single host hiccup must not dominate the number
    e2e_steps = max(args.steps, 2000)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):  # H2D of step k+1 overlaps the kernels of step k
        opt.train_step_host_async(xh, yh, lh)
    ctx.sync()
    t1 = time.perf_counter()
    e2e_s = max_over_ranks(t1 - t0)
    e2e = {"value": gb * e2e_steps / e2e_s, "unit": "samples/s", "steps": e2e_steps,
           "h2d_bytes_per_step": int(x.nbytes + y.nbytes) * world,
           "d2h_bytes_per_step": int(lh.numel() * 4) * world}

    # ---- roofline: eager profiled pass, per-stage CUDA events on the launching stream ----
    ctx.set_profiling(True)
    for _ in range(args.profile_steps):
        flush.zero_()
        opt.train_step(xt, yt, loss, use_graph=False)
    prof = ctx.profile()
    ctx.set_profiling(False)
    hbm, peak_src = peaks()
    stages = {k: {"ms": v["ms"] / v["count"], "gbs": (v["bytes"] / v["count"]) / (v["ms"] / v["count"] * 1e6),
                  "tflops": (v["flops"] / v["count"]) / (v["ms"] / v["count"] * 1e9)}
              for k, v in prof.items() if v["count"]}
    dom = max(prof, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    dom_ms = d["ms"] / d["count"]
    achieved = (d["bytes"] / d["count"]) / (dom_ms * 1e6)  # GB/s
    # DRAM bytes of the dominant stage from the committed ncu --set full capture of the same
    # step (tools/ncu_stages.py), per launch; null when that stage is not in the capture
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{w.name}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        t = tj.get(dom)
        traffic = t["traffic"] if t else None
        if t:
            traffic_src = (f"committed capture {os.path.relpath(tpath, ROOT)} ({tj.get('_source', 'ncu --set full')}); "
                           "not measured in this run")
    hot, full = step_bytes(w, b, materialise)
    eager_step_ms = sum(v["ms"] for v in prof.values()) / args.profile_steps
    ms_per_step = total_ms / args.steps
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "stage_timing": "eager profiled pass (per-stage CUDA events, one stream); value is the graph replay",
                "algorithmic_bytes_per_launch": d["bytes"] / d["count"], "launch_ms": dom_ms,
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)" if peak_src == "measured" else "fallback",
                "step": {"bytes_full": full, "bytes_hot": hot,
                         "frac_full": full / (ms_per_step * 1e6) / hbm,
                         "floor_ms_full": full / (hbm * 1e6)},
                "stages_ms": {k: round(v["ms"], 5) for k, v in sorted(stages.items(), key=lambda kv: -kv[1]["ms"])},
                "eager_stage_sum_ms": eager_step_ms}
    # graph-time stage durations: the same step captured with event-record nodes around every
    # stage (dpg_ctx_set_timeline), replayed, each stage's duration as it overlaps in the graph
    if world == 1:
        tctx = dpg.Context(local)
        tctx.set_timeline(True)
        tm = dpg.Model(tctx, w.layers, w.in_shape, max_batch=b)
        tm.load_params(params)
        to = dpg.DpOptimizer(tm, noise_multiplier=args.sigma, max_grad_norm=args.max_grad_norm,
                             learning_rate=0.1, expected_batch_size=float(gb), noise_seed=3,
                             materialise_grad_sample=materialise)
        for _ in range(5):
            to.train_step(xt, yt, loss)
        tl = tctx.timeline()
        span = max(t0 + dt for _, t0, dt, _ in tl) if tl else 0.0
        roofline["graph_stages_ms"] = {nm: round(dt, 5) for nm, t0, dt, _ in sorted(tl, key=lambda r: -r[2])}
        roofline["graph_timeline"] = {
            "span_ms": round(span, 5),
            "note": "one replay with an event-record node around every stage (PDL edges split at "
                    "stage boundaries, so the span exceeds ms_per_step); durations include the "
                    "overlap with concurrent branches; profiles/r02_timeline_cifar_b512.txt charts it"}
        del to, tm, tctx

    # ---- strong scaling, BASELINE configs[4]: global batch 4096 split over the ranks ----
    strong = None
    if not args.no_strong and w.name == "cifar_b512" and 4096 % world == 0:
        w5 = WORKLOADS["cifar_b4096"]
        from paper_2109_12298_b200.sharding import shard_range
        lo5, hi5 = shard_range(w5.batch, world, rank)  # contiguous sample shard of ONE global batch
        per5 = hi5 - lo5
        p5, x5, y5 = synth(w5, w5.batch)
        x5, y5 = x5[lo5:hi5], y5[lo5:hi5]
        m5 = dpg.Model(ctx, w5.layers, w5.in_shape, max_batch=per5)
        m5.load_params(p5)
        o5 = dpg.DpOptimizer(m5, noise_multiplier=args.sigma, max_grad_norm=args.max_grad_norm,
                             learning_rate=0.1, expected_batch_size=float(w5.batch), noise_seed=3,
                             materialise_grad_sample=materialise)
        ex5 = setup_exchange(o5, exchange) if world > 1 else None
        x5t, y5t = torch.from_numpy(x5).cuda(), torch.from_numpy(y5).cuda()
        l5 = torch.zeros(per5, device="cuda")
        for _ in range(max(3, args.warmup)):
            o5.train_step(x5t, y5t, l5)
        steps5 = max(20, min(args.steps, 200))
        ev5 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps5)]
        barrier()
        torch.cuda.synchronize()
        for i in range(steps5):
            flush.zero_()
            ev5[i][0].record(stream)
            o5.train_step(x5t, y5t, l5)
            ev5[i][1].record(stream)
        torch.cuda.synchronize()
        barrier()
        ctx.sync()
        t5 = max_over_ranks(sum(a.elapsed_time(c) for a, c in ev5))
        strong = {"workload": "cifar_b4096", "scaling": "strong", "global_batch": w5.batch, "per_rank_batch": per5,
                  "n_gpus": world, "steps": steps5, "value": w5.batch * steps5 / (t5 / 1000.0), "unit": "samples/s",
                  "ms_per_step": t5 / steps5, "exchange": ex5,
                  "timing": "device (CUDA events), max over ranks, L2 flushed before every step"}
        del o5, m5

    line = {
        "metric": METRICS.get(w.name, METRIC), "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_for(w.name, gb, b, world, {
            "arm": "B200 (libdpg.so, CUDA graph per step)",
            "exchange": None if world == 1 else (
                "clipped sums summed over peer memory inside the update kernel" if exchange == "p2p"
                else "1 NCCL all-reduce of the clipped sum (+ status lane)"),
            "ranks_share_devices": bool(shared),
            "sigma": args.sigma, "max_grad_norm": args.max_grad_norm,
            "materialise_grad_sample": materialise,
            "clipped_sum": "record pass 2" if (args.csum_from_record and materialise) else "(s.B)^T A",
            "l2": "256 MiB flush before every timed step (outside the step's events)"}),
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": clk,
    }
    if strong:
        line["strong_scaling_cfg5"] = strong
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier()


if __name__ == "__main__":
    main()
