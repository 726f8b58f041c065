"""Several contexts in one process, driven from concurrent host threads (dpg.h: one context per
(host thread, GPU)): the per-(device, function) launch attribute records, the tensor-map encoder
and the cluster-occupancy cache are shared, mutex-guarded state. Two threads running full CIFAR
steps at once — eager and graph-captured — must each produce exactly the single-threaded result."""
import threading

import numpy as np
import pytest

import oracle
from paper_2109_12298_b200.configs import WORKLOADS

pytestmark = pytest.mark.gpu


def _run(w, params, x, y, b, use_graph, out, key):
    import torch
    from paper_2109_12298_b200 import dpg
    ctx = dpg.Context(0)
    m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
    m.load_params(params)
    o = dpg.DpOptimizer(m, noise_multiplier=1.0, max_grad_norm=1.0, learning_rate=0.1,
                        expected_batch_size=float(b), noise_seed=5)
    xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    yt = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32)).cuda()
    for _ in range(3):
        o.train_step(xt, yt, use_graph=use_graph)
    ctx.sync()
    out[key] = m.store_params()


@pytest.mark.parametrize("use_graph", [False, True])
def test_two_contexts_on_two_host_threads(use_graph):
    w = WORKLOADS["cifar_b512"]
    b = 16
    params, x, y = oracle.synth_inputs(w, b=b)
    ref = {}
    _run(w, params, x, y, b, use_graph, ref, "single")
    got = {}
    ts = [threading.Thread(target=_run, args=(w, params, x, y, b, use_graph, got, k)) for k in ("a", "b")]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert set(got) == {"a", "b"}, "a thread failed"
    assert np.array_equal(got["a"], ref["single"]) and np.array_equal(got["b"], ref["single"])
