"""The persistent single-kernel step (csrc/persist.cu) against the oracle and
against the multi-kernel step it replaces for small batches.

dpg_train_step takes it, when enabled (DPG_PERSIST=1), for small conv / linear models (MNIST CNN
b = 64 here); it is opt-in because it measured slower than the multi-kernel step. Reference entry points:
grad_sample.hpp:328-343, optimizer.hpp:62-133, 256-271."""
import os

import numpy as np
import pytest

import oracle
from conftest import maxscaled_err
from paper_2109_12298_b200.configs import WORKLOADS, params_meta

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _persist_on(monkeypatch):
    """The persistent step is opt-in (DPG_PERSIST=1, read per call by dpg_train_step)."""
    monkeypatch.setenv("DPG_PERSIST", "1")


def _run(ctx, w, b, sigma, c, persist, graph=False, steps=1, injected=None):
    import torch
    from paper_2109_12298_b200 import dpg
    params, x, y = oracle.synth_inputs(w, b=b)
    m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
    m.load_params(params)
    o = dpg.DpOptimizer(m, noise_multiplier=sigma, max_grad_norm=c, learning_rate=0.1, expected_batch_size=float(b),
                        noise_seed=3)
    if injected is not None:
        o.set_injected_noise(torch.from_numpy(injected).cuda())
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    loss = torch.zeros(b, device="cuda")
    for _ in range(steps):
        if persist:
            o.train_step(xt, yt, loss, use_graph=graph)
        else:
            o.zero_grad()
            o.forward_backward(xt, yt, loss)
            o.step()
    ctx.sync()
    norms, scales, nclip = o.last_clip_summary()
    return dict(params0=params, x=x, y=y, params=m.store_params(), loss=loss.cpu().numpy(),
                rec=o.grad_sample().cpu().numpy(), summed=o.summed_grad().cpu().numpy(), norms=np.asarray(norms),
                nclip=nclip, launches=ctx.kernel_launches)


@pytest.mark.parametrize("c", [1.0, 2.4])
def test_persist_step_matches_oracle(ctx, c):
    w, b = WORKLOADS["mnist_b64"], 64
    dev = _run(ctx, w, b, 0.0, c, persist=True)
    r64 = oracle.restatement().dpsgd_step(w.layers, w.in_shape, dev["params0"].astype(np.float64),
                                          dev["x"].astype(np.float64), dev["y"].astype(np.float64), 0.0, c, 0.1,
                                          float(b), noise_seed=3)
    np.testing.assert_allclose(dev["loss"], r64["loss"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dev["norms"], r64["norms"], rtol=1e-5)
    assert dev["nclip"] == r64["num_clipped"]
    for (li, k, pname, shape, numel, off) in params_meta(w.layers):
        e = maxscaled_err(dev["rec"][b * off: b * (off + numel)], r64["record"][b * off: b * (off + numel)])
        assert e <= 1e-5, f"record layer {li} {pname}: {e:.3e}"
        e = maxscaled_err(dev["summed"][off:off + numel], r64["summed"][off:off + numel])
        assert e <= 1e-5, f"summed layer {li} {pname}: {e:.3e}"
    e = maxscaled_err(dev["params"].astype(np.float64) - dev["params0"], r64["params"] - dev["params0"])
    assert e <= 1e-5


def test_persist_clipped_sum_is_the_reference_order(ctx):
    """Given the record, the persistent step's clipped sum is the reference's pass 2 bit for bit
    (n ascending, fp32 multiply then add, optimizer.hpp:99-114)."""
    w, b = WORKLOADS["mnist_b64"], 64
    dev = _run(ctx, w, b, 0.0, 2.4, persist=True)
    s = np.asarray(dev["norms"])
    scale = (2.4 / np.maximum(s, 2.4)).astype(np.float32)
    for (li, k, pname, shape, numel, off) in params_meta(w.layers):
        g = dev["rec"][b * off: b * (off + numel)].reshape(b, numel)
        acc = np.zeros(numel, dtype=np.float32)
        for n in range(b):
            acc = (acc + scale[n] * g[n]).astype(np.float32)
        np.testing.assert_array_equal(dev["summed"][off:off + numel], acc)


def test_persist_equals_multikernel_with_noise(ctx):
    """sigma = 1: the same Philox noise (seed, step, element) as the multi-kernel step, so the
    two paths agree to summation order; graph replays equal eager launches bit for bit; one
    launch per step."""
    w, b = WORKLOADS["mnist_b64"], 64
    before = ctx.kernel_launches
    pe = _run(ctx, w, b, 1.0, 1.0, persist=True, steps=3)
    assert pe["launches"] - before == 3, "one kernel per persistent step"
    pg = _run(ctx, w, b, 1.0, 1.0, persist=True, graph=True, steps=3)
    np.testing.assert_array_equal(pe["params"], pg["params"])
    os.environ["DPG_PERSIST"] = "0"
    mk = _run(ctx, w, b, 1.0, 1.0, persist=True, steps=3)  # train_step on the multi-kernel path
    os.environ["DPG_PERSIST"] = "1"
    e = maxscaled_err(pe["params"].astype(np.float64) - pe["params0"], mk["params"].astype(np.float64) - mk["params0"])
    assert e <= 2e-5, f"persistent vs multi-kernel after 3 noisy steps: {e:.3e}"


def test_persist_reports_bad_target(ctx):
    import torch
    from paper_2109_12298_b200 import dpg
    w, b = WORKLOADS["mnist_b64"], 64
    params, x, y = oracle.synth_inputs(w, b=b)
    y = y.copy()
    y[5] = 10.0  # k = 10 classes
    m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
    m.load_params(params)
    o = dpg.DpOptimizer(m, noise_multiplier=0.0, max_grad_norm=1.0, learning_rate=0.1, expected_batch_size=float(b))
    o.train_step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), use_graph=False)
    with pytest.raises(dpg.ParameterError):
        ctx.sync()
    np.testing.assert_array_equal(m.store_params(), params)  # the step must not update
