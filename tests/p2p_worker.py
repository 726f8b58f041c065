"""One rank of the peer-memory exchange test (test_gpu_p2p.py); run as a subprocess.

usage: python p2p_worker.py RANK WORLD PORT OUT_NPZ [ragged|nan]
Every rank takes its contiguous slice of each step's batch (SURVEY.md §8e partitioning), swaps
peer handles over a gloo group, and runs STEPS train steps (the first eager, the rest CUDA-graph
replays) with the exchange inside step(). Writes its final parameters and last summed gradient.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

STEPS = 3
PER_RANK = 24


def problem(world):
    """Deterministic model, parameters and batches shared by the workers and the single-process run."""
    from paper_2109_12298_b200.configs import CIFAR_LAYERS, param_count
    g = np.random.default_rng(7)
    L = param_count(CIFAR_LAYERS)
    params = (0.05 * g.standard_normal(L)).astype(np.float32)
    b = PER_RANK * world
    xs = [g.standard_normal((b, 3, 32, 32)).astype(np.float32) for _ in range(STEPS)]
    ys = [g.integers(0, 10, b).astype(np.float32) for _ in range(STEPS)]
    return CIFAR_LAYERS, (3, 32, 32), params, xs, ys


# ragged shards of the 2-rank batches (48 samples): step 1 leaves rank 1 empty (noise-only
# step_empty_batch there, optimizer.hpp:197-213, while rank 0 steps all 48 samples)
RAGGED = [(30, 18), (48, 0), (20, 28)]


def shard(s, rank, world, total, ragged):
    if not ragged:
        per = total // world
        return rank * per, (rank + 1) * per
    cuts = [0, RAGGED[s][0], total] if world == 2 else [0, total]
    return cuts[rank], cuts[rank + 1]


def run(rank, world, data_world, handles_fn=None, ragged=False, nan=False):
    """Train STEPS steps on rank `rank`'s slice of the data_world-sized batches; world = 1 is the
    single-process run on the full batch. nan: rank 1's input of step 1 holds a NaN — every rank
    must raise for that step and leave its parameters untouched (returned as `errors`)."""
    import torch
    from paper_2109_12298_b200 import dpg
    layers, in_shape, params, xs, ys = problem(data_world)
    total = xs[0].shape[0]
    ctx = dpg.Context(0)
    m = dpg.Model(ctx, layers, in_shape, max_batch=total if ragged else total // world)
    m.load_params(params)
    o = dpg.DpOptimizer(m, noise_multiplier=1.0, max_grad_norm=1.0, learning_rate=0.1,
                        expected_batch_size=float(total), noise_seed=11)
    if handles_fn:
        o.set_peers(rank, handles_fn(o.peer_handle()))
    errors = []
    for s in range(STEPS):
        a, b = shard(s, rank, world, total, ragged)
        if b == a:
            o.zero_grad()
            o.step_empty_batch()
            continue
        xn = xs[s][a:b].copy()
        if nan and s == 1 and rank == 1:
            xn[0, 0, 5, 5] = np.nan
        x = torch.from_numpy(xn).cuda()
        y = torch.from_numpy(ys[s][a:b]).cuda()
        before = m.store_params() if nan else None
        o.train_step(x, y, torch.zeros(b - a, device="cuda"), use_graph=s > 0)
        if nan:
            try:
                o.last_clip_summary()
                errors.append("")
            except dpg.NumericError as e:
                errors.append(str(e))
                assert np.array_equal(m.store_params(), before), "an errored step must not update"
    ctx.sync()
    if nan:
        return m.store_params(), errors
    return m.store_params(), o.summed_grad().cpu().numpy().copy()


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    ragged = len(sys.argv) > 5 and sys.argv[5] == "ragged"
    nan = len(sys.argv) > 5 and sys.argv[5] == "nan"
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def gather(h):
        hs = [None] * world
        dist.all_gather_object(hs, h)
        return hs

    if nan:
        p, errors = run(rank, world, world, gather, nan=True)
        np.savez(out, params=p, errors=np.array(errors))
    else:
        p, summed = run(rank, world, world, gather, ragged)
        np.savez(out, params=p, summed=summed)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
