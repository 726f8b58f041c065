"""Timeline of one TMA-fed convolution launch inside the CIFAR step (trace build of libdpg).

  make -C paper_2109_12298_b200/csrc EXTRA=-DDPG_TG_TRACE OBJ=$PWD/paper_2109_12298_b200/csrc/build_trace \
       OUT=$PWD/paper_2109_12298_b200/libdpg_trace.so
  DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=k python tools/tg_trace_step.py

Runs eager steps; the k-th TMA-fed launch of the process is traced (one step has 6 on CIFAR:
fwd conv2, conv3, conv4, dgrad conv4, conv3, conv2; the first step is launches 0-5). Prints CTA 0's per-stage stamps (producer issue, stage landed, converted, MMA start) and per-tile
(accumulator handed to the epilogue, epilogue done), ns from the first issue."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2109_12298_b200 import dpg  # noqa: E402
from paper_2109_12298_b200.configs import WORKLOADS  # noqa: E402

w = WORKLOADS["cifar_b512"]
b = w.batch
params, x, y = bench.synth(w, b)
ctx = dpg.Context(0)
m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
m.load_params(params)
o = dpg.DpOptimizer(m, noise_multiplier=1.0, max_grad_norm=1.0, learning_rate=0.1, expected_batch_size=float(b))
xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
o.train_step(xt, yt, use_graph=False)
ctx.sync()
lib = dpg.lib()
buf = (ctypes.c_ulonglong * (10 * 256))()
lib.dpg_tg_trace_read(buf)
tr = np.frombuffer(buf, dtype=np.uint64).reshape(10, 256).astype(np.int64)
t0 = tr[0, 0]
print(f"launch {os.environ.get('DPG_TG_TRACE_AT')} cta {os.environ.get('DPG_TG_TRACE_CTA', '0')} "
      f"(t0 = {t0 % 10**9} ns); it: issue landed converted mma_start (ns)")
for i in range(256):
    if tr[0, i] == 0 or (i > 0 and tr[0, i] < t0):
        break
    print(f"{i:3d}: {tr[0, i] - t0:7d} {tr[1, i] - t0:7d} {tr[2, i] - t0:7d} {tr[3, i] - t0:7d}")
for j in range(4):
    if tr[4, j] > 0:
        print(f"tile {j}: tfull {tr[4, j] - t0} epi_done {tr[5, j] - t0}")
        print("   chunks (loaded, split-K exchange, stored):",
              [(int(tr[6, j * 8 + c] - t0), int(tr[8, j * 8 + c] - t0) if tr[8, j * 8 + c] > 0 else None,
                int(tr[7, j * 8 + c] - t0) if tr[7, j * 8 + c] >= t0 else None)
               for c in range(8) if tr[6, j * 8 + c] > 0])
