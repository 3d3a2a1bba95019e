"""Runs the C++ host-API parity driver (tests/cpp/test_engine.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_engine_api():
    exe = os.path.join(ROOT, "tests", "cpp", "test_engine")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1210_4090_b200"), "tests"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout


def test_cpp_driver_builds():
    """The C++ API compiles and links against the library (no GPU needed)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1210_4090_b200"), "tests"], check=True)
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "test_engine"))
