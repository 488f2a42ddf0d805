"""The reference's OWN unit tests (proj/tests/test_synapse.cpp, test_gate.cpp, unmodified)
compiled against the B200 library's cortex:: drop-in (include/cortex/*.hpp +
libcortex_b200.so) instead of the reference's cortex_core, run on the GPU.
Built by `make -C oracle reftests` (needs /root/reference at build time; the
binary travels in oracle/_ref/)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

@pytest.mark.parametrize("name", ["test_synapse", "test_gate"])
def test_reference_unit_tests_pass_on_b200(name):
    """proj/tests/<name>.cpp, unmodified, against the cortex:: drop-in."""
    BIN = os.path.join(ROOT, "oracle", "_ref", name + "_b200")
    if not os.path.exists(BIN):
        pytest.skip(f"oracle/_ref/{name}_b200 not built")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout
