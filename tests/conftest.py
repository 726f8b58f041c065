import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def maxscaled_err(got, ref):
    """max|got - ref| / max|ref| — the per-tensor parity metric."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    if den == 0.0:
        return float(np.abs(got - ref).max()) if ref.size else 0.0
    return float(np.abs(got - ref).max() / den)


@pytest.fixture(scope="session")
def oracle_r():
    import oracle
    return oracle.restatement()


@pytest.fixture(scope="session")
def oracle_ref():
    import oracle
    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return oracle.reference()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2109_12298_b200 import dpg
    return dpg.Context(0)
