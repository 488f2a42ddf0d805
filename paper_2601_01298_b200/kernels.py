"""cortex::kernels on the path (proj/include/cortex/kernels.hpp:31-42):
softmax(), argmax(), attend().

All run on the GPU: softmax in fp64 with the reference's sequential sum (within
1e-15 relative: CUDA vs glibc exp), argmax with the lowest index winning ties,
attend with fp64 accumulation (the reference's own 1e-6, test_kernels.cpp:159-160).
"""
from __future__ import annotations

import numpy as np

import ctypes as C

from ._lib import c_f32p, c_f64p, check, lib, ptr


def attend(q, keys, values, n_entries: int, n_heads: int, d_k: int) -> np.ndarray:
    """kernels.hpp:40-42: returns out (d_model floats)."""
    dm = n_heads * d_k
    qq = np.ascontiguousarray(q, np.float32).reshape(-1)
    kk = np.ascontiguousarray(keys, np.float32).reshape(-1)
    vv = np.ascontiguousarray(values, np.float32).reshape(-1)
    if qq.size != dm or kk.size < n_entries * dm or vv.size < n_entries * dm:
        raise ValueError("attend: q/keys/values sizes do not match n_entries * n_heads * d_k")
    out = np.empty(dm, np.float32)
    check(lib.cx_attend(ptr(qq, c_f32p), ptr(kk, c_f32p), ptr(vv, c_f32p), int(n_entries), int(n_heads), int(d_k),
                        ptr(out, c_f32p)), "attend")
    return out


def softmax(scores) -> np.ndarray:
    """kernels.hpp:31-32 (both overloads: float input is widened, kernels.cpp:89-92)."""
    a = np.asarray(scores)
    n = int(a.size)
    out = np.empty(max(n, 1), np.float64)
    if a.dtype == np.float32:
        aa = np.ascontiguousarray(a, np.float32).reshape(-1)
        check(lib.cx_softmax_f32(ptr(aa, c_f32p), n, ptr(out, c_f64p)), "softmax")
    else:
        aa = np.ascontiguousarray(a, np.float64).reshape(-1)
        check(lib.cx_softmax(ptr(aa, c_f64p), n, ptr(out, c_f64p)), "softmax")
    return out[:n]


def argmax(v) -> int:
    """kernels.hpp:35: lowest index of the maximum."""
    vv = np.ascontiguousarray(v, np.float32).reshape(-1)
    out = C.c_int()
    check(lib.cx_argmax(ptr(vv, c_f32p), int(vv.size), C.byref(out)), "argmax")
    return int(out.value)
