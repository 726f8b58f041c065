"""One eager (non-graph) CIFAR b=512 DP-SGD step for ncu: every kernel of the step launched once
after a warm-up step. Usage: ncu ... python tools/prof_step.py [workload] [batch]"""
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
m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
m.load_params(params)
o = dpg.DpOptimizer(m, noise_multiplier=1.0, max_grad_norm=1.0, learning_rate=0.1, expected_batch_size=float(b))
xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for _ in range(2):
    o.train_step(xt, yt, use_graph=False)
ctx.sync()
torch.cuda.profiler.start()
o.train_step(xt, yt, use_graph=False)
ctx.sync()
torch.cuda.profiler.stop()
print("launches", ctx.kernel_launches)
