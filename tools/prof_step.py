"""One eager (non-graph) CIFAR b=512 DP-SGD step for ncu: every kernel of the step launched once
after a warm-up step. Usage: ncu ... python tools/prof_step.py [workload] [batch]"""
import json
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
# the profiled step runs with stage profiling on: one stream, and the stage sequence (name, kernels)
# is written next to the ncu output so tools/ncu_stages.py can attribute each launch to its stage
ctx.set_profiling(True)
torch.cuda.profiler.start()
o.train_step(xt, yt, use_graph=False)
ctx.sync()
torch.cuda.profiler.stop()
prof = ctx.profile()
ctx.set_profiling(False)
seq = sorted(((v["seq"], k, v["kernels"]) for k, v in prof.items()))
os.makedirs("gpurun_out", exist_ok=True)
with open(os.path.join("gpurun_out", f"stages_{name}.json"), "w") as f:
    json.dump([{"stage": k, "kernels": n, "bytes": prof[k]["bytes"], "flops": prof[k]["flops"]}
               for _, k, n in seq], f, indent=1)
print("launches", ctx.kernel_launches)
