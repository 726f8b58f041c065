"""Generate tests/golden/*.npz from the REAL reference (oracle/_ref/libdpgref.so).

TEST INFRASTRUCTURE ONLY. Run in the container where /root/reference exists:
    make -C oracle && python oracle/make_golden.py
The fixtures pin the restatement (tests/test_golden.py, CPU) and the device step (GPU) on boxes
where the reference tree is absent. Inputs are produced with the reference's own RngStream /
build_model (SURVEY.md §8(d) seeds: model 1, data 2, targets 3, noise 3).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from paper_2109_12298_b200.configs import LayerDesc as L, WORKLOADS, Workload  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

SMALL_EMBED = Workload("embed_small", (L.embedding(50, 8), L.flatten(), L.linear(96, 2)), (12,), 3, 2,
                       tokens=50, description="embedding 50x8 + linear, T=12")

CASES = [
    # name, workload, b, sigma, C, shards
    ("mnist_b4", WORKLOADS["mnist_b64"], 4, 1.0, 1.0, None),
    ("mnist_b4_c2.4", WORKLOADS["mnist_b64"], 4, 1.0, 2.4, None),
    ("cifar_b3_c1.5", WORKLOADS["cifar_b512"], 3, 1.0, 1.5, None),
    ("cifar_b4_shards", WORKLOADS["cifar_b512"], 4, 1.0, 1.5, [1, 3]),
    ("embed_small_b3", SMALL_EMBED, 3, 1.0, 1.0, None),
]


def main():
    ref = oracle.reference()
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "rng_seed3.npz"), u64=ref.u64(3, 1000), normal=ref.normals(3, 1000),
                        below=ref.below(3, 1000, 10000), gaussian_f32=ref.gaussian(3, 1000, 1.7))
    for name, w, b, sigma, c, shards in CASES:
        p, x, y = oracle.synth_inputs(w, b=b, impl=ref)
        r = ref.dpsgd_step(w.layers, w.in_shape, p, x, y, sigma, c, 0.1, float(b), noise_seed=3, shards=shards)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), params=p, x=x, y=y, sigma=sigma, c=c, lr=0.1,
                            expected_batch=float(b),
                            shards=np.array(shards if shards else [b], dtype=np.int64),
                            **{f"out_{k}": v for k, v in r.items() if isinstance(v, np.ndarray)},
                            out_num_clipped=r["num_clipped"])
        print("wrote", name)


if __name__ == "__main__":
    main()
