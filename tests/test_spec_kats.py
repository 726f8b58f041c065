"""SPEC known-answer tests and properties (SPEC.md:51-53, 62, 189-191, 203, 211, 274-294,
310-314) on the oracle restatement — the reference ships no tests, so these prose KATs are its
test suite. CPU only."""
import math

import numpy as np
import pytest

import oracle
from paper_2109_12298_b200.configs import LayerDesc as L, Workload


def test_batched_outer_kats(oracle_r):
    # n=1, b=(1,0), a=(2,3) -> [[2,3],[0,0]]
    gw, gb = oracle_r.rule_linear(np.array([[[2, 3]]], np.float32), np.array([[[1, 0]]], np.float32))
    assert np.array_equal(gw[0], [[2, 3], [0, 0]])
    # annihilator
    gw, _ = oracle_r.rule_linear(np.zeros((2, 3, 4), np.float32), np.ones((2, 3, 5), np.float32))
    assert not gw.any()
    # n=3, middle 4 vs loop, rel 1e-6
    g = np.random.default_rng(0)
    a, h = g.standard_normal((3, 4, 6)), g.standard_normal((3, 4, 5))
    gw, gb = oracle_r.rule_linear(a, h)
    ref = np.einsum("nmi,nmj->nij", h, a)
    assert np.abs(gw - ref).max() <= 1e-12 * np.abs(ref).max()
    np.testing.assert_allclose(gb, h.sum(1), rtol=1e-12)


def test_linear_unit_highway_kat(oracle_r):
    # 1x2 linear, unit highway, x1=(1,2), x2=(3,4) -> per-sample grads (1,2), (3,4)
    gw, _ = oracle_r.rule_linear(np.array([[[1, 2]], [[3, 4]]], np.float32), np.ones((2, 1, 1), np.float32))
    assert np.array_equal(gw.reshape(2, 2), [[1, 2], [3, 4]])


def test_identical_samples_identical_grads(oracle_r):
    # b identical samples -> identical per-sample grads; mean == batch grad
    w = Workload("t", (L.linear(5, 4), L.relu(), L.linear(4, 3)), (5,), 4, 3)
    p, x, y = oracle.synth_inputs(w, b=1, dtype=np.float64)
    x4, y4 = np.repeat(x, 4, 0), np.repeat(y, 4, 0)
    r = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x4, y4, 0.0, 1e9, 0.1, 4.0)
    rec = oracle.record_split(r["record"], w.layers, 4)
    for t in rec:
        assert np.array_equal(t[0], t[1]) and np.array_equal(t[0], t[3])


def test_embedding_kats(oracle_r):
    # single token -> one nonzero row; repeated token -> summed rows; == one-hot matmul
    idx = np.array([[2, 2, 0]], np.float64)
    hw = np.array([[[1, 1], [2, 3], [5, 7]]], np.float64)
    out = oracle_r.rule_embedding(idx, hw, 4)[0]
    assert np.array_equal(out, [[5, 7], [0, 0], [3, 4], [0, 0]])
    onehot = np.eye(4)[idx[0].astype(int)]
    assert np.array_equal(out, onehot.T @ hw[0])


def test_conv_identity_kernel(oracle_r):
    # 1x1 identity-kernel case; zero input -> zero
    x = np.arange(18, dtype=np.float64).reshape(2, 1, 3, 3)
    gw, gb = oracle_r.rule_conv2d(x, np.ones((2, 1, 3, 3)), 1, 1, 1, 0)
    assert np.array_equal(gw.reshape(2), x.reshape(2, -1).sum(1))
    gw, _ = oracle_r.rule_conv2d(np.zeros_like(x), np.ones((2, 1, 3, 3)), 1, 1, 1, 0)
    assert not gw.any()


def test_clip_kats(oracle_r):
    # g1=(3,0), g2=(0,0.5), C=1 -> sum (1, 0.5)
    s, n, sc, k = oracle_r.clip_and_sum([np.array([[3.0, 0.0], [0.0, 0.5]])], 1.0)
    assert np.array_equal(s[0], [1.0, 0.5]) and k == 1
    # all N <= C -> plain sum
    g = np.random.default_rng(1).standard_normal((7, 5)) * 0.1
    s, n, sc, k = oracle_r.clip_and_sum([g], 10.0)
    assert np.array_equal(sc, np.ones(7)) and k == 0
    np.testing.assert_allclose(s[0], g.sum(0), rtol=1e-12)


def test_post_clip_norm_invariant_and_monotone(oracle_r):
    # ||scale_i g_i|| <= C(1+1e-6); scale monotone in N
    g = np.random.default_rng(2)
    for _ in range(50):
        grads = [g.standard_normal((9, 4)) * g.uniform(0.1, 5), g.standard_normal((9, 3))]
        c = g.uniform(0.5, 3)
        s, n, sc, k = oracle_r.clip_and_sum(grads, c)
        flat = np.concatenate([x.reshape(9, -1) for x in grads], 1)
        assert np.all(np.linalg.norm(flat * sc[:, None], axis=1) <= c * (1 + 1e-6))
        order = np.argsort(n)
        assert np.all(np.diff(sc[order]) <= 0)


def test_noise_kats(oracle_r):
    # sigma=0 identity; fixed seed reproducible; empirical std within 2% of sigma*C
    s = np.random.default_rng(3).standard_normal(100000)
    assert np.array_equal(oracle_r.add_noise(s, 0.0, 1.0, 5), s)
    a = oracle_r.add_noise(s, 1.5, 2.0, 5)
    assert np.array_equal(a, oracle_r.add_noise(s, 1.5, 2.0, 5))
    assert abs((a - s).std() / 3.0 - 1) < 0.02
    # 1e6 draws, mean +-0.005, var +-0.01
    z = oracle_r.gaussian(11, 1_000_000, 1.0, np.float64)
    assert abs(z.mean()) < 0.005 and abs(z.var() - 1) < 0.01


def test_degenerate_dp_is_sgd(oracle_r):
    # sigma=0, C >= max N, E=b -> plain SGD on the mean gradient
    w = Workload("t", (L.linear(6, 4), L.relu(), L.linear(4, 3)), (6,), 5, 3)
    p, x, y = oracle.synth_inputs(w, b=5, dtype=np.float64)
    r = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 0.0, 1e12, 0.1, 5.0)
    mean = np.concatenate([t.reshape(5, -1).mean(0) for t in oracle.record_split(r["record"], w.layers, 5)])
    np.testing.assert_allclose(r["params"], p - 0.1 * mean, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("parts", [[64], [32, 32], [16] * 4, [8] * 8])
def test_virtual_step_partition_invariance(oracle_r, parts):
    # logical 64 as {1x64, 2x32, 4x16, 8x8} -> identical update (fp64, 1e-6)
    w = Workload("t", (L.linear(6, 4), L.relu(), L.linear(4, 3)), (6,), 64, 3)
    p, x, y = oracle.synth_inputs(w, b=64, dtype=np.float64)
    base = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 0.7, 0.1, 64.0)
    r = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 0.7, 0.1, 64.0, shards=parts)
    np.testing.assert_allclose(r["params"], base["params"], rtol=1e-6, atol=1e-12)


def test_record_element_count(oracle_r):
    # record element count == b * L exactly
    from paper_2109_12298_b200.configs import WORKLOADS, param_count
    w = WORKLOADS["mnist_b64"]
    p, x, y = oracle.synth_inputs(w, b=3)
    r = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 1.0, 0.1, 3.0)
    assert r["record"].size == 3 * param_count(w.layers) == 3 * 26010


def test_parameter_errors(oracle_r):
    w = Workload("t", (L.linear(3, 2),), (3,), 2, 2)
    p, x, y = oracle.synth_inputs(w, b=2)
    for bad in (dict(sigma=-1.0), dict(c=0.0), dict(lr=0.0), dict(e=0.0)):
        kw = dict(sigma=1.0, c=1.0, lr=0.1, e=2.0)
        kw.update(bad)
        with pytest.raises(oracle.OracleError) as e:
            oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, kw["sigma"], kw["c"], kw["lr"], kw["e"])
        assert e.value.code == 2
