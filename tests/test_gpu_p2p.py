"""The clipped-sum exchange over peer memory (dpg_optimizer_set_peers).

Two ranks as two processes sharing the one GPU of the test box (CUDA IPC within a device; the
same mapping is NVLink P2P across GPUs), each on its half of every batch: after three steps
(one eager, two CUDA-graph replays) both ranks hold bitwise identical parameters and the same
all-rank clipped sum, and they match one process stepping the full batch within the §8c
tolerance (the two halves' partial sums associate differently; the noise is identical).
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import maxscaled_err

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("ragged", [False, True])
def test_peer_exchange_two_ranks_match_single_process(tmp_path, ctx, ragged):
    """ragged: unequal shards, and one step where rank 1 has no samples (step_empty_batch)."""
    sys.path.insert(0, HERE)
    import p2p_worker
    port = _port()
    outs = [str(tmp_path / f"r{r}.npz") for r in range(2)]
    extra = ["ragged"] if ragged else []
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "p2p_worker.py"), str(r), "2", str(port), outs[r]]
                              + extra,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, start_new_session=True)
             for r in range(2)]
    logs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=300)
            logs.append(out.decode(errors="replace")[-3000:])
    finally:
        for p in procs:
            if p.poll() is None:
                os.killpg(p.pid, 9)
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log
    r0, r1 = np.load(outs[0]), np.load(outs[1])
    assert np.array_equal(r0["params"], r1["params"])
    assert np.array_equal(r0["summed"], r1["summed"])
    p_single, s_single = p2p_worker.run(0, 1, 2, ragged=ragged)
    _, _, params0, _, _ = p2p_worker.problem(2)
    assert maxscaled_err(r0["summed"], s_single) <= 1e-5
    assert maxscaled_err(r0["params"] - params0, p_single - params0) <= 1e-5


def test_error_on_one_rank_skips_the_update_on_every_rank(tmp_path, ctx):
    """A NaN input on rank 1 (NumericError there) must stop the update on rank 0 too: the status
    lane travels with the clipped sums, both ranks raise for that step, keep their parameters,
    and stay bitwise identical afterwards (the reference's step throws before any update)."""
    port = _port()
    outs = [str(tmp_path / f"n{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "p2p_worker.py"), str(r), "2", str(port), outs[r],
                               "nan"], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, start_new_session=True)
             for r in range(2)]
    logs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=300)
            logs.append(out.decode(errors="replace")[-3000:])
    finally:
        for p in procs:
            if p.poll() is None:
                os.killpg(p.pid, 9)
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log
    r0, r1 = np.load(outs[0]), np.load(outs[1])
    e0, e1 = list(r0["errors"]), list(r1["errors"])
    assert e0[0] == "" and e1[0] == "" and e0[2] == "" and e1[2] == "", (e0, e1)
    assert "non-finite per-sample gradient" in e1[1], e1
    assert "another rank" in e0[1], e0
    assert np.array_equal(r0["params"], r1["params"])


def test_peer_exchange_argument_errors(ctx):
    from paper_2109_12298_b200 import dpg
    from paper_2109_12298_b200.configs import LayerDesc as L
    m = dpg.Model(ctx, (L.flatten(), L.linear(12, 3)), (3, 2, 2), max_batch=4)
    o = dpg.DpOptimizer(m)
    h = o.peer_handle()
    assert len(h) == 128
    with pytest.raises(dpg.ParameterError):
        o.set_peers(2, [h, h])
    with pytest.raises(dpg.ParameterError):
        o.set_peers(0, [h] * 9)
    m2 = dpg.Model(ctx, (L.flatten(), L.linear(12, 4)), (3, 2, 2), max_batch=4)
    o2 = dpg.DpOptimizer(m2)
    with pytest.raises(dpg.DimensionError):
        o.set_peers(0, [h, o2.peer_handle()])
    o.set_peers(0, [h])  # world 1: exchange off, NCCL-free single rank
