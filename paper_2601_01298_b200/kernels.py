"""cortex::kernels on the path (proj/include/cortex/kernels.hpp): attend().

Runs on the GPU with fp64 accumulation, matching the reference within its own
1e-6 tolerance (test_kernels.cpp:159-160).  matvec/rmsnorm/rope/argmax are
model projections, out of scope.
"""
from __future__ import annotations

import numpy as np

from ._lib import c_f32p, check, lib, ptr


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
