"""The reference's OWN unit tests (proj/tests/test_synapse.cpp, test_gate.cpp,
test_kernels.cpp, test_model.cpp, test_injector.cpp -- unmodified) compiled against the
B200 library's cortex:: drop-in (include/cortex/*.hpp + libcortex_b200.so) instead of
the reference's cortex_core, run on the GPU.  test_model / test_injector link the
reference's own serial oracle ref::forward_sequence (src/ref/ref_model.cpp): forward_step,
encode_thought and inject on the device must match it (incremental == full recompute
within 1e-6, river logits after an injection == the inline-construction oracle).
Built by `make -C oracle reftests` (needs /root/reference at build time; the
binary travels in oracle/_ref/)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

@pytest.mark.parametrize("name", ["test_synapse", "test_gate", "test_kernels", "test_model", "test_injector"])
def test_reference_unit_tests_pass_on_b200(name):
    """proj/tests/<name>.cpp, unmodified, against the cortex:: drop-in."""
    BIN = os.path.join(ROOT, "oracle", "_ref", name + "_b200")
    if not os.path.exists(BIN):
        pytest.fail(f"oracle/_ref/{name}_b200 not built (make -C oracle reftests)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout


def test_reference_full_unit_suite_on_b200():
    """Every proj/tests/test_*.cpp (synapse, kernels, model, injector, gate, router,
    prism, scheduler, harness), unmodified, linked against the drop-in plus the
    reference sources it does not replace (scheduler, prism, router, audit, harness,
    ref_model) -- the CMake swap of INTEGRATION.md §2."""
    BIN = os.path.join(ROOT, "oracle", "_ref", "unit_b200")
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/unit_b200 not built (make -C oracle reftests)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "failed: 0" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


def test_reference_acceptance_on_b200():
    """proj/tests/acceptance.cpp (AC1-AC9, incl. AC3 landmark fidelity, AC4 hybrid vs
    random, AC5 referential-injection equivalence <= 1e-6 against ref::forward_sequence),
    unmodified, on the drop-in: exits with the number of failed criteria."""
    BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/acceptance_b200 not built (make -C oracle reftests)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200, cwd=os.path.join(ROOT, "oracle", "_ref"))
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "FAIL" not in r.stdout
