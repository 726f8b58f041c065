import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2109_12298_b200 import dpg
ctx = dpg.Context(0)
m, n, k = 128, 32, 32
a = np.zeros((m, k), np.float32); b = np.zeros((n, k), np.float32)
a[np.arange(m), np.arange(m) % k] = 1.0      # A row i selects k = i % 32
b[:, :] = np.arange(n)[:, None] * 100 + np.arange(k)[None, :]   # B[n][k] = 100 n + k
d = dpg.tg_gemm_selftest(ctx, torch.from_numpy(a).cuda(), torch.from_numpy(np.ascontiguousarray(b.T)).cuda(), 32, -32)
ctx.sync()
got = d.cpu().numpy(); ref = a @ b.T
print("ref[0:3,0:6]\n", ref[0:3, 0:6]); print("got[0:3,0:6]\n", got[0:3, 0:6])
print("got rows 8..10\n", got[8:11, 0:6])
print("nonzero", np.count_nonzero(got), "of", got.size)
