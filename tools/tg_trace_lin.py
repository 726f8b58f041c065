"""Timeline of one TMA-fed T > 1 linear launch (tg_linear.cu) at cfg2's shape (trace build).

  make -C paper_2109_12298_b200/csrc EXTRA=-DDPG_TG_TRACE OBJ=$PWD/paper_2109_12298_b200/csrc/build_trace \\
       OUT=$PWD/paper_2109_12298_b200/libdpg_trace.so
  DPG_LIB=libdpg_trace.so DPG_TG_TRACE_AT=k python tools/tg_trace_lin.py

Launch 0 = the rule (per-sample gradients), 1 = the clipped sum. Prints CTA 0's per-stage stamps
(producer issue, stage landed, converted, MMA start) and per-tile (accumulator handed to the
epilogue, epilogue done), ns from the first issue; plus the launch's event time."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2109_12298_b200 import dpg  # noqa: E402

b, t, d, r = 256, 64, 512, 512
g = np.random.default_rng(0)
A = torch.from_numpy(g.standard_normal((b, t, d)).astype(np.float32)).cuda()
H = torch.from_numpy(g.standard_normal((b, t, r)).astype(np.float32)).cuda()
ctx = dpg.Context(0)
gw, gb, sw, sb = dpg.per_sample_rule_linear(ctx, A, H)
scale = torch.rand(b, device="cuda")
out = torch.empty(r, d, device="cuda")
dpg.clipped_sum_linear(ctx, A, H, scale, out_w=out, out_b=torch.empty(r, device="cuda"))
ctx.sync()
lib = dpg.lib()
if not hasattr(lib, "dpg_tg_lin_trace_read"):  # plain build (e.g. under ncu): no timeline
    sys.exit(0)
buf = (ctypes.c_ulonglong * (10 * 256))()
lib.dpg_tg_lin_trace_read(buf)
tr = np.frombuffer(buf, dtype=np.uint64).reshape(10, 256).astype(np.int64)
t0 = tr[0, 0]
print(f"launch {os.environ.get('DPG_TG_TRACE_AT')} cta {os.environ.get('DPG_TG_TRACE_CTA', '0')}; "
      "it: issue landed converted mma_start (ns)")
for i in range(min(256, 64)):
    if tr[0, i] == 0 or (i > 0 and tr[0, i] < t0):
        break
    print(f"{i:3d}: {tr[0, i] - t0:7d} {tr[1, i] - t0:7d} {tr[2, i] - t0:7d} {tr[3, i] - t0:7d}")
for j in range(24):
    if tr[4, j] > 0:
        print(f"tile {j}: tfull {tr[4, j] - t0} epi_done {tr[5, j] - t0}  chunks (loaded, stored):",
              [(int(tr[6, j * 8 + c] - t0), int(tr[7, j * 8 + c] - t0)) for c in range(8)
               if j * 8 + c < 256 and tr[7, j * 8 + c] >= t0])
