"""Time the TMA-fed GEMM core alone (dpg_tg_gemm_selftest) on conv-like shapes (GPU box): the
main loop (long K) and the epilogue's store stream (short K, wide output)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_12298_b200 import dpg  # noqa: E402

ctx = dpg.Context(0)
for (m, n, k, bn, bk) in [(32768, 64, 288, 64, 32), (32768, 64, 288, 64, 16), (32768, 32, 256, 32, 32),
                          (131072, 32, 32, 32, 32), (8192, 64, 576, 32, 32), (32768, 64, 4096, 64, 32),
                          # store-bound: short K, wide output
                          (131072, 64, 16, 64, 16), (65536, 128, 32, 128, 32), (65536, 256, 32, 128, 32)]:
    a = torch.randn(m, k, device="cuda")
    b = torch.randn(n, k, device="cuda")
    for _ in range(3):
        dpg.tg_gemm_selftest(ctx, a, b, bn, bk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dpg.tg_gemm_selftest(ctx, a, b, bn, bk)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    fl = 2 * m * n * k * 3
    gb = 4 * (m * k + n * k * ((m + 127) // 128) + m * n)
    print(f"M={m} N={n} K={k} bn={bn} bk={bk}: {us:7.1f} us  {fl / us / 1e6:7.1f} TFLOP/s(3xTF32 eq)  "
          f"{gb / us / 1e3:7.1f} GB/s  (output {4 * m * n / us / 1e3:7.1f} GB/s)")
