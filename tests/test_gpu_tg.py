"""The TMA-fed tcgen05 GEMM core (csrc/tg_gemm.cuh) on its own: D = A B^T against fp64.

Every convolution contraction of the step is built on this core (TMA boxes -> in-place 3xTF32
split -> tcgen05.mma -> TMEM epilogue), so its numerics are pinned here on plain row-major
operands, with ragged M / N / K (TMA out-of-bounds fill) and the longest K a convolution of the
step contracts (576). Longer chains are not fp32-faithful: the tensor core's fp32 accumulation
error grows with the chain (K = 4096 measured 2.7e-5 max-scaled), which is why the clipped sums
bound their chains (tc_conv.cu kCsumChain)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k,bn,bk", [
    (128, 64, 32, 64, 32), (300, 100, 200, 64, 32), (300, 100, 200, 32, 16), (257, 130, 576, 128, 32),
    (1000, 32, 64, 32, 32), (64, 64, 16, 64, 16),
    # MN-major B (the clipped sums' NHWC input tiles): chunks of 32 along N, ragged N and K
    (256, 96, 64, 96, -32), (300, 192, 288, 192, -32), (128, 64, 32, 64, -32), (200, 100, 100, 96, -32)])
def test_tg_gemm_matches_fp64(ctx, m, n, k, bn, bk):
    import torch
    from paper_2109_12298_b200 import dpg
    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    bt = np.ascontiguousarray(b.T) if bk < 0 else b  # bk < 0: B lands MN-major from [k][n]
    d = dpg.tg_gemm_selftest(ctx, torch.from_numpy(a).cuda(), torch.from_numpy(bt).cuda(), bn, bk)
    ctx.sync()
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    got = d.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    # fp32-faithful to the parity criterion (SURVEY.md §8c, 1e-5 max-scaled): the split operands are
    # exact to 2^-22, but the tensor core's fp32 accumulation adds ~2.5e-8 of max|D| per MMA of the
    # chain (3 K / 8 of them: 5.3e-6 measured at K = 576)
    assert err < 1e-5, f"max-scaled error {err:.3e}"
    # and no bias: mean signed error tiny relative to the spread
    assert abs((got - ref).mean()) < 1e-6 * np.abs(ref).max()


@pytest.mark.parametrize("m,n,k,bn,ck", [
    (256, 64, 288, 64, 2), (300, 64, 576, 64, 4), (128, 32, 64, 32, 2),
    # fewer K blocks (3) than cluster ranks: one rank contributes an empty accumulator
    (1000, 64, 96, 64, 4),
    # more tiles than co-resident clusters: the reduction buffers cycle through several phases
    (25600, 64, 576, 64, 2), (25600, 32, 256, 32, 4)])
def test_tg_gemm_cluster_split_k(ctx, m, n, k, bn, ck):
    """K blocks split over a thread-block cluster, partials summed through distributed shared
    memory in rank order (tg_gemm.cuh): fp64 parity and bitwise determinism across runs."""
    import torch
    from paper_2109_12298_b200 import dpg
    rng = np.random.default_rng(7 * m + n + k + ck)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    d = dpg.tg_gemm_selftest_split(ctx, at, bt, bn, ck)
    d2 = dpg.tg_gemm_selftest_split(ctx, at, bt, bn, ck)
    ctx.sync()
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    got = d.cpu().numpy().astype(np.float64)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-5, f"max-scaled error {err:.3e}"
    assert torch.equal(d, d2), "split-K result differs between runs"
