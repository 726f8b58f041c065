"""Phase timeline of the persistent small-batch step (trace build: EXTRA=-DDPG_PERSIST_TRACE).

  DPG_LIB=libdpg_ptrace.so python tools/persist_trace.py   -> ns per phase of one MNIST b=64 step"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_12298_b200 import dpg  # noqa: E402
from paper_2109_12298_b200.configs import WORKLOADS  # noqa: E402

w = WORKLOADS["mnist_b64"]
params, x, y = bench.synth(w, 64)
ctx = dpg.Context(0)
m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=64)
m.load_params(params)
o = dpg.DpOptimizer(m, noise_multiplier=1.0, max_grad_norm=1.0, learning_rate=0.1, expected_batch_size=64.0)
xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
buf = (ctypes.c_ulonglong * 32)()
for it in range(3):
    dpg.lib().dpg_persist_trace_read(buf)
    o.train_step(xt, yt, use_graph=False)
    ctx.sync()
dpg.lib().dpg_persist_trace_read(buf)
t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
names = ["samples", "factors", "csum"]
prev = t[31]
for i, nm in enumerate(names):
    print(f"{nm:8s} {t[i] - prev:8d} ns")
    prev = t[i]
