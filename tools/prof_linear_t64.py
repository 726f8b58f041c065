"""One cfg2 step (per_sample_rule_linear + clip + clipped sum + noise on A, B [256, 64, 512]) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2109_12298_b200 import dpg  # noqa: E402

ctx = dpg.Context(0)
b, t, d, r = 256, 64, 512, 512
A = torch.randn(b, t, d, device="cuda")
B = torch.randn(b, t, r, device="cuda")
for _ in range(2):
    gw, gb, sw, sb = dpg.per_sample_rule_linear(ctx, A, B)
    norms, scale, _ = dpg.clip_factors(ctx, torch.stack([sw, sb]), 1.0)
    dpg.clipped_sum_linear(ctx, A, B, scale)
ctx.sync()
torch.cuda.profiler.start()
gw, gb, sw, sb = dpg.per_sample_rule_linear(ctx, A, B)
norms, scale, _ = dpg.clip_factors(ctx, torch.stack([sw, sb]), 1.0)
dpg.clipped_sum_linear(ctx, A, B, scale)
ctx.sync()
torch.cuda.profiler.stop()
