"""The C++ example links against the C ABI only (CPU check: the binary exists and resolves libdpg)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_example_links_libdpg():
    exe = os.path.join(ROOT, "paper_2109_12298_b200", "dpg_train")
    assert os.path.exists(exe), "build() compiles examples/dpg_train.cpp"
    ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libdpg.so" in ldd and "not found" not in ldd.split("libdpg.so")[1].splitlines()[0]
