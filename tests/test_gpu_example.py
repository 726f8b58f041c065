"""The C++ host path with no Python in the process: examples/dpg_train.cpp (built next to
libdpg.so by the csrc Makefile) trains the CIFAR CNN through the C ABI with CUDA-graph steps."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2109_12298_b200", "dpg_train")

pytestmark = pytest.mark.gpu


def test_cpp_training_loop():
    if not os.path.exists(BIN):
        pytest.fail("paper_2109_12298_b200/dpg_train missing: run __graft_entry__.build()")
    out = subprocess.run([BIN, "20", "64", "1.0", "1.0"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["finite"] and res["samples_per_s"] > 0 and res["batch"] == 64
    assert 0.0 < res["mean_loss"] < 20.0
