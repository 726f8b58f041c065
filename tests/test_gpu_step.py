"""The whole DP-SGD step on the device (engine ABI) against the oracle's full step.

Inputs are generated exactly as SURVEY.md §8(d) pins them (build_model / gaussian / below with
seeds 1, 2, 3). The device step is compared with the oracle's fp64 step on the same fp32
inputs (per-tensor max-scaled error <= 1e-5) and with its fp32 step (and within 50x the reference's
own fp32 error + 5e-6). Noise is checked three ways:
sigma = 0, injection of the oracle's own noise tensor (mt19937_64 + Box-Muller), and the Philox
distribution test in test_gpu_rules.py.
"""
import numpy as np
import pytest

import oracle
from conftest import maxscaled_err
from paper_2109_12298_b200.configs import WORKLOADS, params_meta

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _n(t):
    return t.detach().cpu().numpy()


def _setup(ctx, name, b, **opt):
    from paper_2109_12298_b200 import dpg
    w = WORKLOADS[name]
    params, x, y = oracle.synth_inputs(w, b=b)
    m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=max(b, 64))
    m.load_params(params)
    cfg = dict(noise_multiplier=0.0, max_grad_norm=1.0, learning_rate=0.1, expected_batch_size=float(b),
               noise_seed=3)
    cfg.update(opt)
    o = dpg.DpOptimizer(m, **cfg)
    return w, params, x, y, m, o, cfg


def _oracle_step(w, params, x, y, cfg, dtype, **kw):
    R = oracle.restatement()
    return R.dpsgd_step(w.layers, w.in_shape, params.astype(dtype), x.astype(dtype), y.astype(dtype),
                        cfg["noise_multiplier"], cfg["max_grad_norm"], cfg["learning_rate"],
                        cfg["expected_batch_size"], noise_seed=cfg["noise_seed"], **kw)


def _cmp(got, r32, r64, name, tol=TOL):
    e = maxscaled_err(got, r64)
    e32 = maxscaled_err(r32, r64)
    assert e <= tol, f"{name}: {e:.3e} vs fp64 (reference fp32 itself: {e32:.3e})"
    assert e <= 50 * e32 + 5e-6, f"{name}: {e:.3e} vs reference fp32 error {e32:.3e}"


@pytest.mark.parametrize("name,b,c", [("mnist_b64", 16, 1.0), ("mnist_b64", 16, 2.4),
                                      ("cifar_b512", 16, 1.0), ("cifar_b512", 16, 1.5),
                                      ("embed_b512", 6, 132.0)])
def test_step_matches_oracle(ctx, name, b, c):
    w, params, x, y, m, o, cfg = _setup(ctx, name, b, max_grad_norm=c)
    loss = _t(np.zeros(b))
    o.forward_backward(_t(x), _t(y), loss)
    rec = _n(o.grad_sample())
    o.step()
    norms, scales, nclip = o.last_clip_summary()
    summed = _n(o.summed_grad())
    grad = _n(o.grad())
    p_new = m.store_params()
    r32 = _oracle_step(w, params, x, y, cfg, np.float32)
    r64 = _oracle_step(w, params, x, y, cfg, np.float64)
    np.testing.assert_allclose(_n(loss), r64["loss"], rtol=1e-5, atol=1e-6)
    for (li, k, pname, shape, numel, off) in params_meta(w.layers):
        sl = slice(b * off, b * (off + numel))
        _cmp(rec[sl], r32["record"][sl], r64["record"][sl], f"record layer {li} {pname}")
        _cmp(summed[off:off + numel], r32["summed"][off:off + numel], r64["summed"][off:off + numel],
             f"summed layer {li} {pname}")
    np.testing.assert_allclose(norms, r64["norms"], rtol=TOL)
    assert nclip == r32["num_clipped"] or abs(nclip - r32["num_clipped"]) <= 1
    np.testing.assert_allclose(scales, r64["scales"], rtol=TOL)
    _cmp(grad, r32["grad"], r64["grad"], "grad")
    _cmp(p_new - params, r32["params"] - params, r64["params"] - params, "update")


@pytest.mark.parametrize("name,b", [("cifar_b512", 12), ("embed_b512", 4)])
def test_injected_noise_matches_reference_stream(ctx, name, b):
    """Inject the oracle's own mt19937_64 noise: device params track the reference step."""
    w, params, x, y, m, o, cfg = _setup(ctx, name, b, noise_multiplier=1.0)
    R = oracle.restatement()
    L = m.L
    noise = R.gaussian(cfg["noise_seed"], L, cfg["noise_multiplier"] * cfg["max_grad_norm"])
    o.set_injected_noise(_t(noise))
    o.forward_backward(_t(x), _t(y))
    o.step()
    p_new = m.store_params()
    r32 = _oracle_step(w, params, x, y, cfg, np.float32)  # draws the same stream itself
    r64 = _oracle_step(w, params, x, y, cfg, np.float64, injected_noise=noise.astype(np.float64))
    _cmp(p_new - params, r32["params"] - params, r64["params"] - params, "update with injected noise")


def test_philox_noise_statistics_in_step(ctx):
    """sigma > 0 with Philox: the update minus the sigma=0 update is N(0, (sigma C / E lr)^2)."""
    b = 16
    w, params, x, y, m, o, cfg = _setup(ctx, "cifar_b512", b, noise_multiplier=2.0)
    o.forward_backward(_t(x), _t(y))
    o.step()
    noisy = m.store_params()
    m.load_params(params)
    o.zero_grad()
    o.set_noise_multiplier(0.0)
    o.forward_backward(_t(x), _t(y))
    o.step()
    clean = m.store_params()
    z = (clean.astype(np.float64) - noisy) / (cfg["learning_rate"] / b) / (2.0 * cfg["max_grad_norm"])
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1.0) < 0.02, (z.mean(), z.std())


def test_virtual_steps_match_reference(ctx):
    """Logical batch as physical shards (optimizer.hpp:166-174) == the reference's virtual steps."""
    b = 24
    shards = [5, 11, 8]
    w, params, x, y, m, o, cfg = _setup(ctx, "cifar_b512", b, max_grad_norm=1.5)
    r0 = 0
    for i, s in enumerate(shards):
        o.forward_backward(_t(x[r0:r0 + s]), _t(y[r0:r0 + s]))
        if i < len(shards) - 1:
            o.virtual_step()
        r0 += s
    assert o.accumulated_samples() == sum(shards[:-1])
    o.step()
    assert o.accumulated_samples() == b
    summed = _n(o.summed_grad())
    p_new = m.store_params()
    r32 = _oracle_step(w, params, x, y, cfg, np.float32, shards=shards)
    r64 = _oracle_step(w, params, x, y, cfg, np.float64, shards=shards)
    _cmp(summed, r32["summed"], r64["summed"], "summed over virtual steps")
    _cmp(p_new - params, r32["params"] - params, r64["params"] - params, "update")
    # and == the single physical batch, up to fp32 reassociation
    r1 = _oracle_step(w, params, x, y, cfg, np.float64)
    assert maxscaled_err(summed, r1["summed"]) <= TOL


def test_lifecycle_errors(ctx):
    from paper_2109_12298_b200 import dpg
    b = 4
    w, params, x, y, m, o, cfg = _setup(ctx, "mnist_b64", b)
    with pytest.raises(dpg.LifecycleError, match="no accumulated samples"):
        o.step()
    with pytest.raises(dpg.LifecycleError, match="virtual_step without a fresh grad_sample"):
        o.virtual_step()
    o.forward_backward(_t(x), _t(y))
    with pytest.raises(dpg.LifecycleError, match="never consumed"):
        o.forward_backward(_t(x), _t(y))
    with pytest.raises(dpg.LifecycleError, match="gradients pending"):
        o.step_empty_batch()
    o.step()
    with pytest.raises(dpg.LifecycleError, match="step called twice"):
        o.step()
    with pytest.raises(dpg.LifecycleError, match="still present"):
        o.forward_backward(_t(x), _t(y))
    o.zero_grad()
    o.zero_grad()  # idempotent
    assert o.summed_grad() is None and o.grad() is None
    with pytest.raises(dpg.LifecycleError):
        o.step()


def test_step_empty_batch_is_noise_only(ctx):
    b = 4
    w, params, x, y, m, o, cfg = _setup(ctx, "mnist_b64", b)
    o.step_empty_batch()  # sigma = 0: parameters unchanged (zero sums, no noise)
    assert np.array_equal(m.store_params(), params)
    assert not _n(o.summed_grad()).any()


def test_nonfinite_input_raises_numeric_and_keeps_params(ctx):
    from paper_2109_12298_b200 import dpg
    b = 8
    w, params, x, y, m, o, cfg = _setup(ctx, "cifar_b512", b)
    x = x.copy()
    x[5, 0, 3, 3] = np.nan
    o.forward_backward(_t(x), _t(y))
    o.step()
    with pytest.raises(dpg.NumericError, match=r"non-finite per-sample gradient in layer \d+ parameter '(weight|bias)' \(sample 5\)"):
        o.last_clip_summary()
    assert np.array_equal(m.store_params(), params)


def test_bad_target_raises_parameter(ctx):
    from paper_2109_12298_b200 import dpg
    b = 4
    w, params, x, y, m, o, cfg = _setup(ctx, "mnist_b64", b)
    y = y.copy()
    y[2] = 10.0
    o.forward_backward(_t(x), _t(y))
    with pytest.raises(dpg.ParameterError, match=r"target class .* \(sample 2\)"):
        ctx.sync()


def test_model_shape_errors(ctx):
    from paper_2109_12298_b200 import dpg
    from paper_2109_12298_b200.configs import LayerDesc as L
    with pytest.raises(dpg.DimensionError, match="expected trailing extent 5"):
        dpg.Model(ctx, [L.linear(5, 2)], (4,), 8)
    with pytest.raises(dpg.DimensionError, match="kernel larger than padded input"):
        dpg.Model(ctx, [L.conv2d(1, 2, 5, 5), L.flatten(), L.linear(2, 2)], (1, 3, 3), 8)
    with pytest.raises(dpg.RegistryError, match="custom"):  # a kind without a device rule
        dpg.Model(ctx, [L(7), L.linear(4, 2)], (4,), 8)
    m = dpg.Model(ctx, [L.linear(4, 3)], (4,), 8)
    o = dpg.DpOptimizer(m)
    with pytest.raises(dpg.DimensionError, match="exceeds"):
        o.forward_backward(_t(np.zeros((9, 4))), _t(np.zeros(9)))
    with pytest.raises(dpg.ParameterError, match="max grad norm"):
        dpg.DpOptimizer(m, max_grad_norm=0.0)


def test_graph_replay_equals_eager(ctx):
    import torch
    b = 32
    w, params, x, y, m, o, cfg = _setup(ctx, "cifar_b512", b, noise_multiplier=1.0)
    xt, yt = _t(x), _t(y)
    loss = torch.zeros(b, device="cuda")
    for _ in range(3):
        o.train_step(xt, yt, loss, use_graph=False)
    eager = m.store_params()
    m.load_params(params)
    from paper_2109_12298_b200 import dpg
    o2 = dpg.DpOptimizer(m, **cfg)
    for _ in range(3):
        o2.train_step(xt, yt, loss, use_graph=True)
    ctx.sync()
    assert np.array_equal(m.store_params(), eager), "graph replay must be bit-identical to eager"
    # replays advance the Philox step on the device; an eager step in between must resynchronise it
    m.load_params(params)
    o5 = dpg.DpOptimizer(m, **cfg)
    for graph in (True, False, True):
        o5.train_step(xt, yt, loss, use_graph=graph)
    ctx.sync()
    assert np.array_equal(m.store_params(), eager), "graph / eager / graph must equal three eager steps"
    # host-buffer path == device path
    m.load_params(params)
    o3 = dpg.DpOptimizer(m, **cfg)
    lh = np.zeros(b, dtype=np.float32)
    for _ in range(3):
        o3.train_step_host(np.ascontiguousarray(x, dtype=np.float32), np.ascontiguousarray(y, dtype=np.float32), lh)
    assert np.array_equal(m.store_params(), eager)
    assert np.all(np.isfinite(lh))
    # pipelined host path (two staging slots, copies on a second stream) == device path,
    # with a different input per step so a slot mix-up would show
    xs = [np.ascontiguousarray(x + np.float32(0.01 * k), dtype=np.float32) for k in range(4)]
    yc = np.ascontiguousarray(y, dtype=np.float32)
    m.load_params(params)
    o4 = dpg.DpOptimizer(m, **cfg)
    for k in range(4):
        o4.train_step(_t(xs[k]), yt, loss, use_graph=True)
    ctx.sync()
    ref = m.store_params()
    m.load_params(params)
    o5 = dpg.DpOptimizer(m, **cfg)
    xh = [torch.from_numpy(a).pin_memory() for a in xs]
    yh = torch.from_numpy(yc).pin_memory()  # host buffers stay alive until ctx.sync()
    lhs = [torch.zeros(b).pin_memory() for _ in range(4)]
    for k in range(4):
        o5.train_step_host_async(xh[k], yh, lhs[k])
    ctx.sync()
    assert np.array_equal(m.store_params(), ref), "pipelined host steps must equal device steps"
    assert all(np.all(np.isfinite(t.numpy())) for t in lhs)


def test_degenerate_dp_equals_sgd(ctx):
    """sigma = 0, C above every norm, E = b -> plain SGD on the mean gradient."""
    b = 16
    w, params, x, y, m, o, cfg = _setup(ctx, "mnist_b64", b, max_grad_norm=1e6)
    o.forward_backward(_t(x), _t(y))
    rec = _n(o.grad_sample())
    o.step()
    p_new = m.store_params()
    mean_grad = np.zeros(m.L)
    for (li, k, pname, shape, numel, off) in params_meta(w.layers):
        mean_grad[off:off + numel] = rec[b * off:b * (off + numel)].reshape(b, numel).astype(np.float64).mean(0)
    sgd = params - 0.1 * mean_grad
    assert maxscaled_err(p_new - params, sgd - params) < 1e-5


def test_variable_batch_graph_cache_equals_eager(ctx):
    """Poisson-style physical batch sizes: 14 steps over 11 distinct sizes (more than the 8-entry
    graph cache, so executables are updated in place) give the eager path's bits."""
    import torch
    from paper_2109_12298_b200 import dpg
    sizes = [32, 17, 29, 32, 9, 24, 31, 12, 20, 17, 27, 14, 32, 5]
    w, params, x, y, m, o, cfg = _setup(ctx, "cifar_b512", 32, noise_multiplier=1.0, expected_batch_size=24.0)
    xt, yt = _t(x), _t(y)
    bufs = {b: (xt[:b].contiguous(), yt[:b].contiguous(), torch.zeros(b, device="cuda")) for b in set(sizes)}
    for b in sizes:
        o.train_step(*bufs[b], use_graph=False)
    eager = m.store_params()
    m.load_params(params)
    o2 = dpg.DpOptimizer(m, **cfg)
    for b in sizes:
        o2.train_step(*bufs[b], use_graph=True)
    ctx.sync()
    assert np.array_equal(m.store_params(), eager), "graph cache replays must be bit-identical to eager"



def test_nccl_allreduce_in_captured_step(ctx):
    """The multi-GPU data path on one GPU: a one-rank NCCL communicator puts ncclAllReduce of the
    clipped sum into the captured step; sum over one rank is the identity, so the
    update must equal the communicator-free step bit for bit (eager and graph)."""
    import torch
    from paper_2109_12298_b200 import dpg
    b = 16
    w, params, x, y, m, o, cfg = _setup(ctx, "cifar_b512", b, noise_multiplier=1.0)
    xt, yt = _t(x), _t(y)
    loss = torch.zeros(b, device="cuda")
    for _ in range(2):  # the multi-kernel step (train_step may take the persistent kernel at this size)
        o.zero_grad()
        o.forward_backward(xt, yt, loss)
        o.step()
    ctx.sync()
    ref = m.store_params()
    c2 = dpg.Context(0)
    c2.init_comm(1, 0, dpg.Context.nccl_unique_id())
    m2 = dpg.Model(c2, w.layers, w.in_shape, max_batch=64)
    m2.load_params(params)
    o2 = dpg.DpOptimizer(m2, **cfg)
    o2.train_step(xt, yt, loss, use_graph=False)
    o2.train_step(xt, yt, loss, use_graph=True)
    c2.sync()
    assert np.array_equal(m2.store_params(), ref)
    buf = torch.arange(10, dtype=torch.float32, device="cuda")
    c2.allreduce_sum(buf)
    c2.sync()
    assert torch.equal(buf, torch.arange(10, dtype=torch.float32, device="cuda"))


def test_graph_timeline_records_every_stage_and_keeps_the_result():
    """dpg_ctx_set_timeline: the stage scopes of a captured step become event nodes; a replay
    yields a start / duration per stage (non-negative, inside the step, branches overlapping the
    main chain) and the step's result is bit-identical to the graph without the nodes."""
    import torch
    from paper_2109_12298_b200 import dpg
    b = 32
    results = []
    for timeline in (False, True):
        ctx = dpg.Context(0)
        ctx.set_timeline(timeline)
        w, params, x, y, m, o, cfg = _setup(ctx, "cifar_b512", b, noise_multiplier=1.0)
        xt, yt = _t(x), _t(y)
        for _ in range(3):
            o.train_step(xt, yt, use_graph=True)
        ctx.sync()
        results.append(m.store_params())
        if timeline:
            tl = ctx.timeline()
            names = [r[0] for r in tl]
            for stage in ("fwd.conv2d[0]", "dgrad.conv2d[2]", "gs.conv2d[2]", "clip_factors",
                          "csum.conv2d[2]", "noise_update"):
                assert stage in names, (stage, names)
            assert all(t0 >= 0.0 and dt >= 0.0 for _, t0, dt, _ in tl)
            span = max(t0 + dt for _, t0, dt, _ in tl)
            assert 0.0 < span < 50.0, span  # ms
            by = {r[0]: r for r in tl}
            # causal order on the main chain; a rule branch overlaps the dgrad chain
            assert by["clip_factors"][1] >= by["fwd.conv2d[0]"][1] + by["fwd.conv2d[0]"][2]
            assert by["noise_update"][1] >= by["clip_factors"][1]
            assert by["gs.conv2d[4]"][1] < by["dgrad.conv2d[2]"][1] + by["dgrad.conv2d[2]"][2]
    assert np.array_equal(results[0], results[1]), "timeline nodes must not change the step"
