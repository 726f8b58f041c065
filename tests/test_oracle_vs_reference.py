"""Pin the oracle: the C restatement (oracle/dpg_oracle*.c) against the reference compiled from
its own sources (oracle/_ref/libdpgref.so), bit for bit, in fp32 and fp64.

These run on CPU only and are the reason the GPU parity tests may trust the restatement.
"""
import numpy as np
import pytest

import oracle
from paper_2109_12298_b200.configs import WORKLOADS, LayerDesc as L


def test_mt19937_64_check_value(oracle_r):
    # C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64 (seed 5489)
    assert int(oracle_r.u64(5489, 10000)[-1]) == 9981545732273789042


def test_rng_streams_bit_exact(oracle_r, oracle_ref):
    for seed in (0, 1, 3, 2 ** 63 + 5):
        assert np.array_equal(oracle_r.u64(seed, 700), oracle_ref.u64(seed, 700))
        assert np.array_equal(oracle_r.normals(seed, 1001), oracle_ref.normals(seed, 1001))
        assert np.array_equal(oracle_r.below(seed, 500, 10000), oracle_ref.below(seed, 500, 10000))
        assert np.array_equal(oracle_r.gaussian(seed, 999, 2.5), oracle_ref.gaussian(seed, 999, 2.5))


@pytest.mark.parametrize("name", ["mnist_b64", "cifar_b512", "embed_b512"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_build_params_bit_exact(oracle_r, oracle_ref, name, dtype):
    w = WORKLOADS[name]
    assert np.array_equal(oracle_r.build_params(w.layers, 1, dtype), oracle_ref.build_params(w.layers, 1, dtype))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_rules_bit_exact(oracle_r, oracle_ref, dtype):
    g = np.random.default_rng(0)
    a = g.standard_normal((5, 7, 9)).astype(dtype)
    h = g.standard_normal((5, 7, 4)).astype(dtype)
    for x, y in zip(oracle_r.rule_linear(a, h), oracle_ref.rule_linear(a, h)):
        assert np.array_equal(x, y)
    x = g.standard_normal((3, 4, 9, 8)).astype(dtype)
    hw = g.standard_normal((3, 5, 5, 4)).astype(dtype)  # oh = 5, ow = 4
    for p, q in zip(oracle_r.rule_conv2d(x, hw, 3, 3, 2, 1), oracle_ref.rule_conv2d(x, hw, 3, 3, 2, 1)):
        assert np.array_equal(p, q)
    idx = g.integers(0, 6, size=(4, 9)).astype(dtype)
    he = g.standard_normal((4, 9, 3)).astype(dtype)
    assert np.array_equal(oracle_r.rule_embedding(idx, he, 11), oracle_ref.rule_embedding(idx, he, 11))
    grads = [g.standard_normal((6, 5)).astype(dtype), (4 * g.standard_normal((6, 3, 2))).astype(dtype)]
    r1, r2 = oracle_r.clip_and_sum(grads, 1.5), oracle_ref.clip_and_sum(grads, 1.5)
    for s, t in zip(r1[0], r2[0]):
        assert np.array_equal(s, t)
    assert np.array_equal(r1[1], r2[1]) and np.array_equal(r1[2], r2[2]) and r1[3] == r2[3]
    s = g.standard_normal(77).astype(dtype)
    assert np.array_equal(oracle_r.add_noise(s, 1.3, 0.7, 9), oracle_ref.add_noise(s, 1.3, 0.7, 9))


@pytest.mark.parametrize("name,b,c", [("mnist_b64", 8, 1.0), ("mnist_b64", 8, 2.4),
                                      ("cifar_b512", 6, 1.5), ("embed_b512", 3, 132.0)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_full_step_bit_exact(oracle_r, oracle_ref, name, b, c, dtype):
    w = WORKLOADS[name]
    p, x, y = oracle.synth_inputs(w, b=b, dtype=dtype)
    a = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, c, 0.1, float(b))
    r = oracle_ref.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, c, 0.1, float(b))
    for k in a:
        if isinstance(a[k], np.ndarray):
            assert np.array_equal(a[k], r[k]), k
        else:
            assert a[k] == r[k], k


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_virtual_steps_and_injection_bit_exact(oracle_r, oracle_ref, dtype):
    w = WORKLOADS["cifar_b512"]
    b = 9
    p, x, y = oracle.synth_inputs(w, b=b, dtype=dtype)
    a = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 1.5, 0.1, float(b), shards=[2, 3, 4])
    r = oracle_ref.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 1.5, 0.1, float(b), shards=[2, 3, 4])
    for k in ("summed", "grad", "params", "norms", "record"):
        assert np.array_equal(a[k], r[k]), k
    noise = oracle_r.gaussian(3, p.size, 1.5, dtype)
    a = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 1.5, 0.1, float(b), injected_noise=noise)
    r = oracle_ref.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 1.5, 0.1, float(b), injected_noise=noise)
    assert np.array_equal(a["params"], r["params"])
    # injecting the stream the reference draws == letting it draw (noise_seed 3)
    d = oracle_ref.dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 1.5, 0.1, float(b))
    assert np.array_equal(a["params"], d["params"])


def test_vectorized_matches_microbatch_oracle(oracle_r, oracle_ref):
    """Appendix A vs Appendix B: the record equals the micro-batch oracle."""
    w = WORKLOADS["mnist_b64"]
    p, x, y = oracle.synth_inputs(w, b=4, dtype=np.float64)
    a = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 0.0, 1.0, 0.1, 4.0)
    mb = oracle_ref.microbatch_oracle(w.layers, w.in_shape, p, x, y)
    rec = a["record"]
    assert np.abs(rec - mb).max() <= 1e-10 * np.abs(mb).max()


def test_errors_match_reference(oracle_r, oracle_ref):
    w = WORKLOADS["mnist_b64"]
    p, x, y = oracle.synth_inputs(w, b=4)
    xb = x.copy()
    xb[2, 0, 5, 5] = np.nan
    with pytest.raises(oracle.OracleError) as e1:
        oracle_r.dpsgd_step(w.layers, w.in_shape, p, xb, y, 1.0, 1.0, 0.1, 4.0)
    with pytest.raises(oracle.OracleError) as e2:
        oracle_ref.dpsgd_step(w.layers, w.in_shape, p, xb, y, 1.0, 1.0, 0.1, 4.0)
    assert e1.value.code == e2.value.code == 5
    assert e1.value.msg == e2.value.msg
    yb = y.copy()
    yb[1] = 12.0
    with pytest.raises(oracle.OracleError) as e3:
        oracle_ref.dpsgd_step(w.layers, w.in_shape, p, x, yb, 1.0, 1.0, 0.1, 4.0)
    assert e3.value.code == 2 and "target class" in e3.value.msg
    with pytest.raises(oracle.OracleError) as e4:
        oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, yb, 1.0, 1.0, 0.1, 4.0)
    assert e4.value.code == 2


def test_nonparam_models_and_ragged_layers(oracle_r, oracle_ref):
    layers = (L.linear(6, 5, bias=False), L.relu(), L.linear(5, 3))
    from paper_2109_12298_b200.configs import Workload
    w = Workload("t", layers, (6,), 7, 3)
    p, x, y = oracle.synth_inputs(w, b=7, dtype=np.float64)
    a = oracle_r.dpsgd_step(w.layers, w.in_shape, p, x, y, 0.5, 0.8, 0.1, 7.0)
    r = oracle_ref.dpsgd_step(w.layers, w.in_shape, p, x, y, 0.5, 0.8, 0.1, 7.0)
    assert np.array_equal(a["params"], r["params"]) and np.array_equal(a["record"], r["record"])


def test_reference_norm_rules_and_step(oracle_ref):
    """The layer_norm / group_norm rules the GPU parity tests check against (grad_sample.hpp:87-131):
    the reference's fp64 rules are the plain sums, and its step runs a model with both layers."""
    from paper_2109_12298_b200.configs import LayerDesc as L, param_count
    g = np.random.default_rng(5)
    xh, h = g.standard_normal((3, 4, 6)), g.standard_normal((3, 4, 6))
    gg, gb = oracle_ref.rule_norm(xh, h, False)  # layer_norm over the trailing 6
    np.testing.assert_allclose(gg, (xh * h).sum(1), rtol=1e-14)
    np.testing.assert_allclose(gb, h.sum(1), rtol=1e-14)
    gg, gb = oracle_ref.rule_norm(xh, h, True)  # group_norm over [b, 4 channels, 6]
    np.testing.assert_allclose(gg, (xh * h).sum(2), rtol=1e-14)
    layers = (L.conv2d(3, 4, 3, 3, 1, 1), L.group_norm(2, 4), L.relu(), L.flatten(), L.linear(64, 8),
              L.layer_norm(8), L.relu(), L.linear(8, 3))
    p = g.standard_normal(param_count(layers)) * 0.3
    x = g.standard_normal((5, 3, 4, 4))
    y = g.integers(0, 3, 5).astype(np.float64)
    r = oracle_ref.dpsgd_step(layers, (3, 4, 4), p, x, y, 0.0, 1.0, 0.1, 5.0)
    assert np.all(np.isfinite(r["params"])) and np.all(r["norms"] > 0)
