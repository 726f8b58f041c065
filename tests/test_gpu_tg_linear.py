"""The T > 1 linear rule and clipped sum on the TMA-fed core (tg_linear.cu) on both sides of every
shape rule the core has: BK = 16 (T <= 16) and 32, K blocks past T (zero fill of the 3-D tensor
map), d and r not multiples of the 128-wide tile, several tiles per sample, the norms-only rule,
the clipped sum's `accumulate` flag and split counts, and the fallbacks (misaligned operands, and
DPG_TG_LIN=0 in a fresh process) onto the register-gather kernels.

Reference: per_sample_rule_linear grad_sample.hpp:53-59 (batched_outer tensor.hpp:303-338), the
clipped sum optimizer.hpp:99-114. Tolerance as tests/test_gpu_rules.py: max-scaled error vs the
fp64 oracle <= 1e-5 and within 50x the reference's own fp32 error + 5e-6.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import maxscaled_err

pytestmark = pytest.mark.gpu

TOL = 1e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# b, T, d, r
SHAPES = [
    (3, 7, 36, 44),      # BK = 16, one partial K block, d / r below one tile
    (2, 20, 132, 260),   # BK = 32, a partial second K block, 2 x 3 tiles with ragged edges
    (2, 100, 64, 128),   # four K blocks, the last partial
    (5, 64, 512, 512),   # cfg2's per-sample shape
    (40, 16, 96, 80),    # BK = 16 exactly, many samples (clipped-sum splits)
]


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _n(t):
    return t.detach().cpu().numpy()


def _check(got, ref32, ref64, name):
    e_gpu = maxscaled_err(got, ref64)
    e_ref = maxscaled_err(ref32, ref64)
    assert e_gpu <= TOL, f"{name}: gpu vs fp64 {e_gpu:.3e} > {TOL}"
    assert e_gpu <= 50 * e_ref + 5e-6, f"{name}: gpu {e_gpu:.3e} vs reference fp32 {e_ref:.3e}"


def _inputs(b, t, d, r, seed):
    g = np.random.default_rng(seed)
    return g.standard_normal((b, t, d)).astype(np.float32), g.standard_normal((b, t, r)).astype(np.float32)


@pytest.mark.parametrize("shape", SHAPES)
def test_tg_linear_rule(ctx, oracle_r, shape):
    from paper_2109_12298_b200 import dpg
    b, t, d, r = shape
    a, h = _inputs(b, t, d, r, sum(shape))
    gw, gb, sw, sb = dpg.per_sample_rule_linear(ctx, _t(a), _t(h))
    rw32, rb32 = oracle_r.rule_linear(a, h)
    rw64, _ = oracle_r.rule_linear(a.astype(np.float64), h.astype(np.float64))
    _check(_n(gw), rw32, rw64, f"rule {shape}")
    assert np.array_equal(_n(gb), rb32), "bias: sequential double sum, bit-exact"
    gwn = _n(gw).astype(np.float64)
    np.testing.assert_allclose(_n(sw), (gwn ** 2).reshape(b, -1).sum(1), rtol=1e-10)
    # norms only: the same fused norm without the record
    _, _, sw2, sb2 = dpg.per_sample_rule_linear(ctx, _t(a), _t(h), grad=False)
    assert np.array_equal(_n(sw), _n(sw2)) and np.array_equal(_n(sb), _n(sb2))


@pytest.mark.parametrize("shape", SHAPES)
def test_tg_linear_clipped_sum(ctx, oracle_r, shape):
    import torch
    from paper_2109_12298_b200 import dpg
    b, t, d, r = shape
    a, h = _inputs(b, t, d, r, 7 * sum(shape))
    sc = np.random.default_rng(b).uniform(0.1, 1.0, size=b).astype(np.float32)
    sw, sb = dpg.clipped_sum_linear(ctx, _t(a), _t(h), _t(sc))
    ref64 = np.einsum("n,nto,nti->oi", sc.astype(np.float64), h.astype(np.float64), a.astype(np.float64))
    gw32, _ = oracle_r.rule_linear(a, h)
    ref32 = np.zeros((r, d), np.float32)
    for n in range(b):
        ref32 = (ref32 + np.float32(sc[n]) * gw32[n]).astype(np.float32)
    _check(_n(sw), ref32, ref64, f"clipped sum {shape}")
    # accumulate: out += the same sum (virtual steps, optimizer.hpp:240-254)
    base = torch.full((r, d), 0.25, device="cuda")
    dpg.clipped_sum_linear(ctx, _t(a), _t(h), _t(sc), out_w=base, out_b=torch.zeros(r, device="cuda"),
                           accumulate=True)
    _check(_n(base) - 0.25, ref32, ref64, f"clipped sum accumulate {shape}")


def test_tg_linear_misaligned_falls_back(ctx, oracle_r):
    """A 4-byte-offset operand cannot be a TMA tensor map: the register-gather kernel takes it and
    gives the same records within tolerance."""
    import torch
    from paper_2109_12298_b200 import dpg
    b, t, d, r = 3, 20, 64, 48
    a, h = _inputs(b, t, d, r, 11)
    buf = torch.empty(a.size + 1, device="cuda")
    buf[1:] = _t(a).reshape(-1)
    a_off = buf[1:].view(b, t, d)  # 4 bytes past a 256-byte allocation: not 16-byte aligned
    assert a_off.data_ptr() % 16 != 0
    gw, _, sw, _ = dpg.per_sample_rule_linear(ctx, a_off, _t(h))
    gw_al, _, sw_al, _ = dpg.per_sample_rule_linear(ctx, _t(a), _t(h))
    rw32, _ = oracle_r.rule_linear(a, h)
    rw64, _ = oracle_r.rule_linear(a.astype(np.float64), h.astype(np.float64))
    _check(_n(gw), rw32, rw64, "misaligned rule")
    assert maxscaled_err(_n(gw), _n(gw_al).astype(np.float64)) <= 2e-6
    np.testing.assert_allclose(_n(sw), _n(sw_al), rtol=1e-5)


@pytest.mark.parametrize("env", [{"DPG_TG_LIN": "0"}, {"DPG_TG_LIN_BN": "128"}])
def test_tg_linear_alternate_paths(env):
    """Switches read once per process, so in a fresh process: DPG_TG_LIN=0 puts the linear rule /
    clipped sum on the register-gather kernels; DPG_TG_LIN_BN=128 keeps the rule on 128-wide
    double-buffered tiles instead of the 256-wide single-buffered ones."""
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_tg_linear.py"), "-k", "rule or clipped_sum"],
                       env=dict(os.environ, **env), cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("b,c", [(12, 1.0), (12, 50.0)])
def test_tg_linear_in_the_engine(ctx, b, c):
    """A sequence model through the engine: Linear on [b, T, d] (mid = T = 20 > 1, the TMA-fed rule
    and clipped sum), ReLU, a second T > 1 Linear whose input is that ReLU's output (the
    converters' ReLU path), flatten, the classifier. Whole step against the oracle's fp64 step:
    record, norms, clipped sums, update (grad_sample.hpp:277-343, optimizer.hpp:62-133)."""
    import oracle
    from paper_2109_12298_b200 import dpg
    from paper_2109_12298_b200.configs import LayerDesc as L, Workload, params_meta
    layers = (L.linear(64, 96), L.relu(), L.linear(96, 32), L.relu(), L.flatten(), L.linear(20 * 32, 10))
    w = Workload("seq_t20", layers, (20, 64), b, 10)
    params, x, y = oracle.synth_inputs(w, b=b)
    m = dpg.Model(ctx, layers, w.in_shape, max_batch=b)
    m.load_params(params)
    cfg = dict(noise_multiplier=0.0, max_grad_norm=c, learning_rate=0.1, expected_batch_size=float(b), noise_seed=3)
    o = dpg.DpOptimizer(m, **cfg)
    o.forward_backward(_t(x), _t(y))
    rec = _n(o.grad_sample())
    o.step()
    summed = _n(o.summed_grad())
    norms, _, _ = o.last_clip_summary()
    p_new = m.store_params()
    R = oracle.restatement()
    res = {dt: R.dpsgd_step(layers, w.in_shape, params.astype(dt), x.astype(dt), y.astype(dt), 0.0, c, 0.1,
                            float(b), noise_seed=3) for dt in (np.float32, np.float64)}
    r32, r64 = res[np.float32], res[np.float64]
    for (li, k, pname, shape, numel, off) in params_meta(layers):
        sl = slice(b * off, b * (off + numel))
        _check(rec[sl], r32["record"][sl], r64["record"][sl], f"record layer {li} {pname}")
        _check(summed[off:off + numel], r32["summed"][off:off + numel], r64["summed"][off:off + numel],
               f"summed layer {li} {pname}")
    np.testing.assert_allclose(norms, r64["norms"], rtol=TOL)
    e = maxscaled_err(p_new.astype(np.float64) - params, r64["params"] - params)
    assert e <= TOL, f"update: {e:.3e}"


def test_tg_linear_operator_calls_in_a_captured_graph():
    """The T > 1 linear operator calls fork their bias work onto the context's side stream and
    join it back: captured into a CUDA graph on the context's stream and replayed,
    they give the eager results bit for bit (rule + norms, bias rule, clipped sums)."""
    import torch
    from paper_2109_12298_b200 import dpg
    s = torch.cuda.Stream()
    ctx = dpg.Context(0, stream=s)
    b, t, d, r = 6, 20, 64, 96
    a, h = _inputs(b, t, d, r, 5)
    A, H = _t(a), _t(h)
    sc = _t(np.random.default_rng(1).uniform(0.1, 1.0, size=b).astype(np.float32))
    gw, gb, sw, sb = (torch.zeros((b, r, d), device="cuda"), torch.zeros((b, r), device="cuda"),
                      torch.zeros(b, dtype=torch.float64, device="cuda"), torch.zeros(b, dtype=torch.float64, device="cuda"))
    cw, cb = torch.zeros((r, d), device="cuda"), torch.zeros(r, device="cuda")
    lib, P = dpg.lib(), dpg._p

    def calls():
        dpg._check(lib.dpg_grad_sample_linear(ctx.h, P(A), P(H), b, t, d, r, P(gw), P(gb), P(sw), P(sb)), ctx.h)
        dpg._check(lib.dpg_clipped_sum_linear(ctx.h, P(A), P(H), P(sc), b, t, d, r, P(cw), P(cb), 0), ctx.h)

    with torch.cuda.stream(s):
        calls()  # eager: creates the side stream and the workspaces
    ctx.sync()
    eager = [x.clone() for x in (gw, gb, sw, sb, cw, cb)]
    for x in (gw, gb, sw, sb, cw, cb):
        x.zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        calls()
    g.replay()
    torch.cuda.synchronize()
    for x, e, name in zip((gw, gb, sw, sb, cw, cb), eager, ("gw", "gb", "sq_w", "sq_b", "sum_w", "sum_b")):
        assert torch.equal(x, e), f"graph replay differs from the eager call: {name}"
