"""The plain-C consumer (tests/c_consumer/smoke.c) runs on the B200: known-answer
selection through the C ABI, error categories as status codes."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_gpu_c_consumer(tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2601_01298_b200")
    exe = tmp_path / "c_smoke"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(root, "include"), os.path.join(root, "tests", "c_consumer",
                    "smoke.c"), "-L", libdir, "-lcortex_b200", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "idx=0,3" in r.stdout
