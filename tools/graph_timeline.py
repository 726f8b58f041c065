"""Timeline of one CUDA-graph DP-SGD step (dpg_ctx_set_timeline): each stage's start and duration
inside the replayed graph, so the overlap of the branches and the critical path are visible.

    python tools/graph_timeline.py [workload] [batch]

Prints the stages by start time with a bar chart, then the step's span. Event-record nodes split
the PDL edges at stage boundaries, so the span is a little longer than the bench's ms_per_step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2109_12298_b200 import dpg  # noqa: E402
from paper_2109_12298_b200.configs import WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cifar_b512"
w = WORKLOADS[name]
b = int(sys.argv[2]) if len(sys.argv) > 2 else w.batch
params, x, y = bench.synth(w, b)
ctx = dpg.Context(0)
ctx.set_timeline(True)
m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
m.load_params(params)
o = dpg.DpOptimizer(m, noise_multiplier=1.0, max_grad_norm=1.0, learning_rate=0.1, expected_batch_size=float(b))
xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for _ in range(20):
    o.train_step(xt, yt, use_graph=True)
ctx.sync()
tl = sorted(ctx.timeline(), key=lambda r: r[1])
span = max(t0 + dt for _, t0, dt, _ in tl)
scale = 100.0 / span
print(f"{'stage':24s} {'start':>8s} {'dur':>8s}  (us; step span {span * 1e3:.1f} us)")
for nm, t0, dt, k in tl:
    a, l = int(t0 * scale), max(1, int(dt * scale))
    print(f"{nm:24s} {t0 * 1e3:8.1f} {dt * 1e3:8.1f}  {' ' * a}{'#' * l}")
