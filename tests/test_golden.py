"""Golden fixtures generated from the real reference by oracle/make_golden.py.

CPU: the restatement reproduces every fixture bit for bit (this is what pins the oracle on a box
without /root/reference). GPU: the device step lands within the stated tolerance of the fixture.
"""
import glob
import os

import numpy as np
import pytest

import oracle
from conftest import maxscaled_err
from paper_2109_12298_b200.configs import LayerDesc as L, WORKLOADS, Workload

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SMALL_EMBED = Workload("embed_small", (L.embedding(50, 8), L.flatten(), L.linear(96, 2)), (12,), 3, 2, tokens=50)
WL = {"mnist": WORKLOADS["mnist_b64"], "cifar": WORKLOADS["cifar_b512"], "embed": SMALL_EMBED}
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")) if "rng" not in p)


def _load(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return WL[name.split("_")[0]], d


def test_fixtures_present():
    assert len(CASES) >= 5


def test_rng_golden(oracle_r):
    d = np.load(os.path.join(GOLDEN, "rng_seed3.npz"))
    assert np.array_equal(oracle_r.u64(3, 1000), d["u64"])
    assert np.array_equal(oracle_r.normals(3, 1000), d["normal"])
    assert np.array_equal(oracle_r.below(3, 1000, 10000), d["below"])
    assert np.array_equal(oracle_r.gaussian(3, 1000, 1.7), d["gaussian_f32"])


@pytest.mark.parametrize("name", CASES)
def test_restatement_reproduces_golden(oracle_r, name):
    w, d = _load(name)
    shards = [int(s) for s in d["shards"]]
    r = oracle_r.dpsgd_step(w.layers, w.in_shape, d["params"], d["x"], d["y"], float(d["sigma"]),
                            float(d["c"]), float(d["lr"]), float(d["expected_batch"]), noise_seed=3,
                            shards=shards if len(shards) > 1 else None)
    for k in ("record", "summed", "grad", "params", "norms", "scales", "loss", "logits"):
        assert np.array_equal(r[k], d["out_" + k]), k
    assert r["num_clipped"] == int(d["out_num_clipped"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_step_vs_golden(ctx, oracle_r, name):
    """Device step with the reference's own noise injected, vs the reference's fp32 output."""
    import torch
    from paper_2109_12298_b200 import dpg
    w, d = _load(name)
    b = d["x"].shape[0]
    shards = [int(s) for s in d["shards"]]
    m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
    m.load_params(d["params"])
    o = dpg.DpOptimizer(m, noise_multiplier=float(d["sigma"]), max_grad_norm=float(d["c"]),
                        learning_rate=float(d["lr"]), expected_batch_size=float(d["expected_batch"]))
    noise = oracle_r.gaussian(3, m.L, float(d["sigma"]) * float(d["c"]))
    o.set_injected_noise(torch.from_numpy(noise).cuda())
    r0 = 0
    for i, s in enumerate(shards):
        o.forward_backward(torch.from_numpy(d["x"][r0:r0 + s]).cuda(), torch.from_numpy(d["y"][r0:r0 + s]).cuda())
        if i < len(shards) - 1:
            o.virtual_step()
        r0 += s
    o.step()
    summed = o.summed_grad().cpu().numpy()
    p_new = m.store_params()
    p64 = oracle_r.dpsgd_step(w.layers, w.in_shape, d["params"].astype(np.float64), d["x"].astype(np.float64),
                              d["y"].astype(np.float64), float(d["sigma"]), float(d["c"]), float(d["lr"]),
                              float(d["expected_batch"]), injected_noise=noise.astype(np.float64),
                              shards=shards if len(shards) > 1 else None)
    e_gpu = maxscaled_err(summed, p64["summed"])
    e_ref = maxscaled_err(d["out_summed"], p64["summed"])
    assert e_gpu <= 1e-5 and e_gpu <= 50 * e_ref + 5e-6, (e_gpu, e_ref)
    e_gpu = maxscaled_err(p_new - d["params"], p64["params"] - d["params"])
    e_ref = maxscaled_err(d["out_params"] - d["params"], p64["params"] - d["params"])
    assert e_gpu <= 1e-5 and e_gpu <= 50 * e_ref + 5e-6, (e_gpu, e_ref)
