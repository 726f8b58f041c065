"""The C ABI library loads and exports every symbol include/dpg.h declares (CPU, no compute)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dpg.h")
LIB = os.path.join(ROOT, "paper_2109_12298_b200", "libdpg.so")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"DPG_API\s+[\w\s\*]+?\b(dpg_\w+)\s*\(", txt)))


def test_header_declares_the_abi():
    names = declared()
    for must in ("dpg_grad_sample_linear", "dpg_grad_sample_conv2d", "dpg_grad_sample_embedding",
                 "dpg_clip_factors", "dpg_clipped_sum_conv2d", "dpg_noise_update", "dpg_allreduce_sum",
                 "dpg_forward_backward", "dpg_step", "dpg_virtual_step", "dpg_zero_grad"):
        assert must in names
    assert len(names) >= 45


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "libdpg.so not built (run __graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dpg_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    # nothing else leaks (hidden visibility)
    assert exported == set(declared())


def test_python_binding_covers_abi_and_loads():
    from paper_2109_12298_b200 import dpg
    assert set(dpg.exported_symbols()) == set(declared())
    assert dpg.lib().dpg_abi_version() == 2


def test_ctx_create_without_gpu_fails_cleanly():
    import ctypes
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2109_12298_b200 import dpg
    h = ctypes.c_void_p()
    code = dpg.lib().dpg_ctx_create(0, None, ctypes.byref(h))
    assert code == 6 and not h.value  # DPG_ERR_CUDA, no context, no crash
    assert dpg.lib().dpg_last_error(None)


def test_layer_desc_layout_matches_header():
    import ctypes
    from paper_2109_12298_b200.configs import CLayerDesc
    assert ctypes.sizeof(CLayerDesc) == 8 + 12 * 8 + 8  # + norm_size, groups, eps
    assert CLayerDesc.in_features.offset == 8 and CLayerDesc.padding.offset == 80


def test_workspace_queries_on_host():
    """dpg_*_workspace_size (size the arena once, no allocation in hot calls) are
    host-only: sizes for the CIFAR layers, 0 for invalid extents."""
    from paper_2109_12298_b200 import dpg
    conv = (512, 16, 16, 32, 64, 3, 3, 2, 1)  # conv2 of the CIFAR model
    gs = dpg.workspace_size("grad_sample_conv2d", *conv)
    cs = dpg.workspace_size("clipped_sum_conv2d", *conv)
    assert gs >= 8 * 512 and gs % 8 == 0
    assert cs >= 4 * 512 * 64  # at least the per-sample bias sums
    assert dpg.workspace_size("grad_sample_linear", 512, 1, 512, 10) >= 8 * 512
    assert dpg.workspace_size("clipped_sum_linear", 256, 64, 512, 512) > 0
    assert dpg.workspace_size("grad_sample_embedding", 512, 256, 10000, 128) >= 8 * 512 * 256
    assert dpg.workspace_size("clipped_sum_embedding", 512, 256, 10000, 128) > 0
    # invalid extents: 0, no exception across the ABI
    assert dpg.workspace_size("grad_sample_conv2d", 512, 2, 2, 32, 64, 3, 3, 1, 0) == 0  # kernel > input
    assert dpg.workspace_size("grad_sample_conv2d", 4, 8, 8, 0, 4, 3, 3, 1, 1) == 0
    assert dpg.workspace_size("grad_sample_linear", 4, 0, 3, 3) == 0
