"""layer_norm / group_norm on the device against the reference itself.

The C restatement covers the north-star layer kinds only, so these tests use the reference compiled
from its sources (oracle/_ref, the `oracle_ref` fixture): the per-sample rules
(grad_sample.hpp:87-131) must match it bit for bit (sequential fp32 sums in the reference's order),
and a whole DP-SGD step of a model with both layers (conv -> group_norm -> relu -> linear ->
layer_norm -> relu -> linear) must match its fp64 step within the §8c tolerance.
"""
import numpy as np
import pytest

from conftest import maxscaled_err
from paper_2109_12298_b200.configs import LayerDesc as L, param_count, params_meta

pytestmark = pytest.mark.gpu

TOL = 1e-5
LAYERS = (L.conv2d(3, 8, 3, 3, 1, 1), L.group_norm(2, 8), L.relu(), L.flatten(), L.linear(8 * 6 * 6, 32),
          L.layer_norm(32), L.relu(), L.linear(32, 5))
IN_SHAPE = (3, 6, 6)


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _n(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("group,shape", [(False, (5, 7, 48)), (False, (3, 1, 300)), (True, (4, 8, 25)),
                                         (True, (2, 16, 1))])
def test_norm_rules_bit_exact(ctx, oracle_ref, group, shape):
    from paper_2109_12298_b200 import dpg
    g = np.random.default_rng(sum(shape))
    xh = g.standard_normal(shape).astype(np.float32)
    hw = g.standard_normal(shape).astype(np.float32)
    rule = dpg.per_sample_rule_group_norm if group else dpg.per_sample_rule_layer_norm
    gg, gb, sg, sb = rule(ctx, _t(xh), _t(hw))
    rg, rb = oracle_ref.rule_norm(xh, hw, group)
    assert np.array_equal(_n(gg), rg)
    assert np.array_equal(_n(gb), rb)
    np.testing.assert_allclose(_n(sg), (rg.astype(np.float64) ** 2).sum(1), rtol=1e-12)
    np.testing.assert_allclose(_n(sb), (rb.astype(np.float64) ** 2).sum(1), rtol=1e-12)


def _inputs(b, seed=1):
    g = np.random.default_rng(seed)
    p = np.empty(param_count(LAYERS), dtype=np.float32)
    for (li, k, name, shape, numel, off) in params_meta(LAYERS):
        if name == "gamma":
            p[off:off + numel] = 1.0 + 0.3 * g.standard_normal(numel)
        else:
            p[off:off + numel] = 0.3 * g.standard_normal(numel)
    x = g.standard_normal((b,) + IN_SHAPE).astype(np.float32)
    y = g.integers(0, 5, b).astype(np.float32)
    return p, x, y


@pytest.mark.parametrize("b,c", [(6, 1.0), (9, 2.2)])
def test_norm_model_step_matches_reference(ctx, oracle_ref, b, c):
    from paper_2109_12298_b200 import dpg
    params, x, y = _inputs(b)
    m = dpg.Model(ctx, LAYERS, IN_SHAPE, max_batch=16)
    m.load_params(params)
    o = dpg.DpOptimizer(m, noise_multiplier=0.0, max_grad_norm=c, learning_rate=0.1,
                        expected_batch_size=float(b), noise_seed=3)
    loss = _t(np.zeros(b))
    o.forward_backward(_t(x), _t(y), loss)
    rec = _n(o.grad_sample())
    o.step()
    norms, scales, nclip = o.last_clip_summary()
    summed = _n(o.summed_grad())
    p_new = m.store_params()
    r64 = oracle_ref.dpsgd_step(LAYERS, IN_SHAPE, params.astype(np.float64), x.astype(np.float64),
                                y.astype(np.float64), 0.0, c, 0.1, float(b))
    r32 = oracle_ref.dpsgd_step(LAYERS, IN_SHAPE, params, x, y, 0.0, c, 0.1, float(b))
    np.testing.assert_allclose(_n(loss), r64["loss"], rtol=1e-5, atol=1e-6)
    for (li, k, name, shape, numel, off) in params_meta(LAYERS):
        sl = slice(b * off, b * (off + numel))
        e = maxscaled_err(rec[sl], r64["record"][sl])
        e32 = maxscaled_err(r32["record"][sl], r64["record"][sl])
        assert e <= TOL and e <= 50 * e32 + 5e-6, f"record layer {li} {name}: {e:.3e} (ref fp32 {e32:.3e})"
        e = maxscaled_err(summed[off:off + numel], r64["summed"][off:off + numel])
        assert e <= TOL, f"summed layer {li} {name}: {e:.3e}"
    np.testing.assert_allclose(norms, r64["norms"], rtol=TOL)
    np.testing.assert_allclose(scales, r64["scales"], rtol=TOL)
    assert abs(nclip - r32["num_clipped"]) <= 1 if "num_clipped" in r32 else True
    e = maxscaled_err(p_new - params, r64["params"] - params)
    assert e <= TOL, f"update {e:.3e}"


def test_norm_model_graph_replay_and_record_free(ctx, oracle_ref):
    """The captured train step and the non-materialised (norms-only) mode give the same update."""
    import torch
    from paper_2109_12298_b200 import dpg
    b = 8
    params, x, y = _inputs(b, seed=4)
    outs = []
    for mat, graph in [(True, False), (True, True), (False, True)]:
        m = dpg.Model(ctx, LAYERS, IN_SHAPE, max_batch=b)
        m.load_params(params)
        o = dpg.DpOptimizer(m, noise_multiplier=0.0, max_grad_norm=1.0, learning_rate=0.1,
                            expected_batch_size=float(b), materialise_grad_sample=mat)
        o.train_step(_t(x), _t(y), torch.zeros(b, device="cuda"), use_graph=graph)
        ctx.sync()
        outs.append(m.store_params())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_norm_shape_errors(ctx):
    from paper_2109_12298_b200 import dpg
    with pytest.raises(dpg.DimensionError):
        dpg.Model(ctx, (L.flatten(), L.layer_norm(7), L.linear(108, 3)), IN_SHAPE, max_batch=4)
    with pytest.raises(dpg.DimensionError):
        dpg.Model(ctx, (L.group_norm(2, 4), L.flatten(), L.linear(108, 3)), IN_SHAPE, max_batch=4)
