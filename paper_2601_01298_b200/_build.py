"""In-tree build of libcortex_b200.so (sm_100a) with nvcc.

The shared library holds the CUDA kernels, the extern "C" boundary
(include/cortex_b200.h) and the C++ cortex:: drop-in shim (include/cortex/).
It is written next to this file so it travels to the GPU box with the repo.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libcortex_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CU_SOURCES = ["synapse_kernels.cu", "select64.cu", "select128.cu", "select_tc.cu", "attend_kernels.cu", "decode_tc.cu", "capi.cu", "comm.cu", "probe.cu", "forward.cu", "cortex_runtime.cu"]
CPP_SOURCES = ["cortex_api.cpp", "cortex_model.cpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++20",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
    "-I" + INCLUDE, "-I" + CSRC,
] + os.environ.get("CX_NVCC_EXTRA", "").split()  # experiments only (e.g. -DCX_TC_OP_BUFS=2)


def _sources():
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    srcs += [os.path.join(CSRC, s) for s in CPP_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    return srcs


def _deps():
    out = []
    for d in (CSRC, INCLUDE, os.path.join(INCLUDE, "cortex")):
        if os.path.isdir(d):
            out += [os.path.join(d, f) for f in os.listdir(d)]
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps() + [__file__])


NEGCTL_LIB = os.path.join(ROOT, "tests", "negctl", "libcortex_negctl.so")
# test-only variant (tests/test_gpu_decode_scale.py negative control): the decode
# score GEMM without its bf16 lo terms.  Never loaded by the product.
NEGCTL_DEFS = {"decode_tc.cu": ["-DCX_NEGCTL_BF16_S"]}


def _link(objs, out):
    tmp = out + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs + \
          ["-lcudart_static", "-lpthread", "-ldl", "-lrt"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date() and os.path.exists(NEGCTL_LIB):
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(NEGCTL_LIB), exist_ok=True)
    objs, negobjs, cmds = [], [], []
    for src in _sources():
        base = os.path.basename(src)
        obj = os.path.join(objdir, base + ".o")
        if src.endswith(".cu"):
            cmd = [NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj] + (["-Xptxas", "-v"] if verbose else [])
        else:
            cmd = ["g++", "-std=c++20", "-O3", "-fPIC", "-I" + INCLUDE, "-I/usr/local/cuda/include", "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
        objs.append(obj)
        if base in NEGCTL_DEFS:
            nobj = os.path.join(objdir, base + ".negctl.o")
            cmds.append([NVCC] + NVCC_FLAGS + NEGCTL_DEFS[base] + ["-c", src, "-o", nobj])
            negobjs.append(nobj)
        else:
            negobjs.append(obj)
    # translation units compile independently: one nvcc per source, in parallel
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    _link(objs, LIB)
    _link(negobjs, NEGCTL_LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
