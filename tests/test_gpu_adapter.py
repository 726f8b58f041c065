"""Drop-in proof at the reference's own plugin API: the reference engine (compute_grad_samples,
make_private, DpOptimizer — compiled from /root/reference into oracle/_ref/adapter_parity)
driving the GPU GradSampleRules of integration/dpgrad_gpu_rules.hpp, registered with
override_existing = true (grad_sample.hpp:159-167)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_parity")

pytestmark = pytest.mark.gpu


def test_reference_engine_with_gpu_rules():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_parity not built (reference tree absent at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    line = out.stdout.strip().splitlines()[-1]
    res = json.loads(line)
    assert out.returncode == 0, res
    for model in ("mnist", "cifar", "embedding", "norms"):
        assert res[model]["record_maxscaled"] <= 1e-5, res
        assert res[model]["params_maxscaled"] <= 1e-5, res
