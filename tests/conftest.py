import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu on the GPU box")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.load()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.load_ref()
    if r is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return r


@pytest.fixture
def cx_option():
    """Pin a kernel path on the device ctx for one test (cx_ctx_set_option);
    restored afterwards.  Usage: cx_option("select_cluster", 4)."""
    saved = []

    def pin(name, value):
        from paper_2601_01298_b200 import device
        saved.append((name, device.set_option(name, value)))

    yield pin
    from paper_2601_01298_b200 import device
    for name, old in reversed(saved):
        device.set_option(name, old)
