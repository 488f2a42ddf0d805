"""CPU-side checks of the drop-in boundary (no compute calls need a GPU):

* libcortex_b200.so loads and exports every entry point include/cortex_b200.h
  declares, and the ctypes binding covers exactly that set;
* the product contains sm_100a code (cuobjdump) and no CPU fallback: without a
  device a valid compute call returns CX_DEVICE_ERROR;
* validation happens before any device work and maps the reference's checks
  onto the reference's error categories, in the reference's order.
"""
import ctypes as C
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "cortex_b200.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cx_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_01298_b200 import _lib
    return _lib


def test_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 50
    missing = [s for s in syms if not hasattr(lib.lib, s)]
    assert not missing, missing
    assert sorted(lib.EXPORTED_SYMBOLS) == syms


def test_cpp_shim_symbols_exported(lib):
    """The C++ cortex:: drop-in shim lives in the same library."""
    nm = shutil.which("nm")
    if nm is None:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-DC", lib.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ("cortex::select_landmarks_points(", "cortex::attention_scores_points(", "cortex::select_landmarks(",
                "cortex::SynapseBuffer::push(", "cortex::kernels::attend(", "cortex::inject(",
                "cortex::KvCache::append_entry("):
        assert sym in out, sym


def test_library_is_sm100a_only(lib):
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_abi_version_and_launch_counter(lib):
    assert lib.lib.cx_abi_version() == 1
    assert lib.lib.cx_kernel_launch_count() >= 0


def _select(lib, cloud, attn, k, lam):
    idx = np.zeros(max(1, k), np.int64)
    sc = np.zeros(max(1, k), np.float64)
    n = C.c_int64(0)
    c = np.ascontiguousarray(cloud, np.float32)
    a = np.ascontiguousarray(attn, np.float64)
    return lib.lib.cx_select_landmarks_points(c.ctypes.data_as(lib.c_f32p), c.shape[0], c.shape[1],
                                              a.ctypes.data_as(lib.c_f64p), a.size, k, lam,
                                              idx.ctypes.data_as(lib.c_i64p), sc.ctypes.data_as(lib.c_f64p),
                                              C.byref(n))


def test_validation_precedes_device_work(lib):
    cloud = np.zeros((3, 2), np.float32)
    # synapse.cpp:219-223 order: k, then lambda, then attention length
    assert _select(lib, cloud, np.zeros(3), 0, 0.5) == 1           # config_error
    assert _select(lib, cloud, np.zeros(3), 1, 1.5) == 1           # config_error
    assert _select(lib, cloud, np.zeros(3), 0, 7.0) == 1           # k checked first
    assert _select(lib, cloud, np.zeros(2), 1, 0.5) == 5           # precondition_error
    assert _select(lib, cloud, np.zeros(2), 0, 0.5) == 1           # config before precondition
    q = np.zeros(2, np.float32)
    out = np.zeros(3)
    f = lib.lib.cx_attention_scores_points
    P = lambda a, t: a.ctypes.data_as(t)  # noqa: E731
    assert f(P(cloud, lib.c_f32p), 0, 2, P(q, lib.c_f32p), 2, 1, P(out, lib.c_f64p)) == 5  # empty set
    assert f(P(cloud, lib.c_f32p), 3, 2, P(q, lib.c_f32p), 3, 1, P(out, lib.c_f64p)) == 5  # width
    assert f(P(cloud, lib.c_f32p), 3, 2, P(q, lib.c_f32p), 2, 3, P(out, lib.c_f64p)) == 5  # heads
    assert lib.lib.cx_hausdorff_to_subset(P(cloud, lib.c_f32p), 3, 2, None, 0, P(out, lib.c_f64p)) == 5
    assert lib.lib.cx_kvcache_create(2, 2, 8, 3, 16, 4, C.byref(C.c_void_p())) == 1  # n_heads*d_k != d_model


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    st = _select(lib, np.zeros((3, 2), np.float32), np.zeros(3), 2, 0.5)
    assert st == 100  # CX_DEVICE_ERROR
    assert "no CUDA device" in lib.lib.cx_last_error().decode()
    import paper_2601_01298_b200 as cx
    with pytest.raises(cx.errors.device_error):
        cx.select_landmarks_points(np.zeros((3, 2), np.float32), np.zeros(3), 2, 0.5)
    with pytest.raises(cx.errors.config_error):
        cx.select_landmarks_points(np.zeros((3, 2), np.float32), np.zeros(3), 0, 0.5)


def test_host_mirror_logic():
    import paper_2601_01298_b200 as cx
    with pytest.raises(cx.errors.config_error):
        cx.ModelConfig(n_heads=3, d_model=64, d_k=16).validate()
    with pytest.raises(cx.errors.config_error):
        cx.ModelConfig(n_heads=1, d_model=3, d_k=3).validate()
    cx.ModelConfig().validate()
    p = cx.VirtualPositionPlanner(7168, 8192)
    assert p.reserved_start() == 7168 and p.reserve(1000) == 7168 and p.reserve(24) == 8168
    with pytest.raises(cx.errors.capacity_error):
        p.reserve(1)
    with pytest.raises(cx.errors.precondition_error):
        p.reserve(0)
    with pytest.raises(cx.errors.config_error):
        cx.VirtualPositionPlanner(8192, 8192)
    assert cx.InjectionRecord.csv_header() == "thought_id,token_count,virtual_position_base,applied_at_stream_position"
    blk = cx.KvBlock(base_position=1, token_count=2, n_layers=2, d_model=3, keys=np.arange(12, dtype=np.float32))
    assert list(blk.key(1, 0)) == [6, 7, 8]


def test_oracle_is_not_linked_by_the_product(lib):
    """The product never links or imports the checker."""
    nm = shutil.which("nm")
    if nm:
        out = subprocess.run([nm, "-D", lib.LIB_PATH], capture_output=True, text=True).stdout
        assert "orc_" not in out and "ref_select" not in out
    pkg = os.path.join(ROOT, "paper_2601_01298_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in txt and "oracle/" not in txt.replace("oracle/_ref", ""), f


def test_plain_c_consumer_compiles_and_links(tmp_path):
    """include/cortex_b200.h is a C ABI: a C11 program (no C++, no torch) compiles
    warning-free against it and links against libcortex_b200.so.  (Run on the GPU
    in test_gpu_c_consumer.)"""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2601_01298_b200")
    exe = tmp_path / "c_smoke"
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "c_consumer", "smoke.c"), "-L", libdir, "-lcortex_b200",
                        "-Wl,-rpath," + libdir, "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert exe.exists()


def test_release_library_has_no_debug_knobs():
    """The experiment switches (phase tracing, skipping a decode role's math, the
    L1 carveout pad, chunk overrides) are compiled out of the release library
    (-DCX_EXPERIMENTS builds only); path pinning goes through cx_ctx_set_option."""
    from paper_2601_01298_b200 import _lib
    with open(_lib.LIB_PATH, "rb") as f:
        blob = f.read()
    for knob in (b"CX_TC_SKIP", b"CX_TC_TRACE", b"CX_TC_SMEM_PAD", b"CX_SEL_TRACE", b"CX_SEL_DUMP", b"CX_SEL_OCC",
                 b"CX_E2E_CHUNKS", b"CX_SEL_C", b"CX_DECODE", b"CX_TC_PER_LH", b"CX_HOST_UPLOAD_VALUES"):
        assert knob not in blob, knob
