"""Multi-rank host logic on CPU (gloo, world_size 2): each rank clips and sums its contiguous
sample shard, one all-reduce combines the clipped sums, and every rank adds the SAME noise once
from the shared seed and applies the same update — equal to the reference's virtual-step path
with physical batches = rank shards, and identical on both ranks."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2109_12298_b200.configs import WORKLOADS
    from paper_2109_12298_b200.sharding import shard_range
    w = WORKLOADS["cifar_b512"]
    B = 10
    p, x, y = oracle.synth_inputs(w, b=B, dtype=np.float64)
    lo, hi = shard_range(B, world, rank)
    R = oracle.restatement()
    sigma, c, lr = 1.0, 1.5, 0.1
    # local clipped sum of this rank's shard (sigma = 0: the step's summed output is pre-noise)
    part = R.dpsgd_step(w.layers, w.in_shape, p, x[lo:hi], y[lo:hi], 0.0, c, lr, float(B))["summed"]
    t = torch.from_numpy(part.copy())
    dist.all_reduce(t)  # the one collective of the step
    summed = t.numpy()
    # noise once, from the shared seed, then the update (optimizer.hpp:256-271), on every rank
    noised = R.add_noise(summed, sigma, c, seed=3)
    params = p - (noised * (1.0 / B)) * lr
    q.put((rank, params))
    dist.destroy_process_group()


def test_two_rank_shard_allreduce_equals_virtual_steps():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert np.array_equal(res[0], res[1]), "ranks must hold bitwise-identical parameters"
    import oracle
    from paper_2109_12298_b200.configs import WORKLOADS
    w = WORKLOADS["cifar_b512"]
    p, x, y = oracle.synth_inputs(w, b=10, dtype=np.float64)
    ref = oracle.restatement().dpsgd_step(w.layers, w.in_shape, p, x, y, 1.0, 1.5, 0.1, 10.0, shards=[5, 5])
    assert np.abs(res[0] - ref["params"]).max() <= 1e-13


def test_shard_ranges_cover_batch():
    from paper_2109_12298_b200.sharding import shard_range
    for B in (1, 7, 512, 4096):
        for W in (1, 2, 3, 8):
            rs = [shard_range(B, W, r) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [h - l for l, h in rs]
            assert max(sizes) - min(sizes) <= 1


def test_bench_spawns_its_own_ranks_without_torchrun():
    """`python bench.py --gpus 2` (the driver's plain form, no torchrun) re-launches itself as two
    ranks on 127.0.0.1 over gloo; under N > 1 rank 0 alone runs the reference arm and prints ONE
    JSON line with the shared config keys, and every rank exits 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import oracle
    if not (oracle.reference_available(fast=True) or os.path.exists(oracle.RESTATEMENT_SO)):
        pytest.skip("oracle not built")
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--workload", "mnist_b64", "--steps", "1", "--warmup", "0"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert set(line["config"]) == {"workload", "global_batch", "per_rank_batch", "parallelism", "detail"}
    assert line["e2e"]["h2d_bytes_per_step"] == 0
