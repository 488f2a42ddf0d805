"""TEST INFRASTRUCTURE ONLY -- ctypes front-end for the CPU checkers.

Two interchangeable back-ends with one Python surface:

* ``load()``      -> the plain-C restatement (``oracle/build/liboracle.so``,
                     source ``oracle/cortex_oracle.c``; every function cites the
                     reference file:line it restates).
* ``load_ref()``  -> the unmodified reference library compiled from
                     /root/reference sources (``oracle/_ref/libcortex_ref.so``,
                     recipe ``oracle/Makefile``), or ``None`` if not built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / baseline.  The product
package (``paper_2601_01298_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcortex_ref.so")

# Mirrors proj/include/cortex/errors.hpp:10-41 (and cx_status in include/cortex_b200.h).
STATUS_NAMES = {
    1: "config_error",
    2: "capacity_error",
    3: "topology_error",
    4: "sequencing_error",
    5: "precondition_error",
    6: "cap_error",
    7: "degenerate_input_error",
    99: "std_exception",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        self.kind = STATUS_NAMES.get(code, f"status_{code}")
        super().__init__(f"{where}: {self.kind}")


_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ct)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


class _OrcRng(C.Structure):
    _fields_ = [("state", C.c_uint64), ("spare", C.c_double), ("has_spare", C.c_int)]


class Rng:
    """cortex::Rng (rng.hpp:11-48) on either back-end."""

    def __init__(self, backend: "Backend", seed: int):
        self._b = backend
        if backend.is_ref:
            self._h = C.c_void_p(backend.lib.ref_rng_new(C.c_uint64(seed)))
        else:
            self._s = _OrcRng()
            backend.lib.orc_rng_init(C.byref(self._s), C.c_uint64(seed))

    def __del__(self):
        if getattr(self, "_b", None) is not None and self._b.is_ref and getattr(self, "_h", None):
            self._b.lib.ref_rng_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h if self._b.is_ref else C.byref(self._s)

    def next_u64(self) -> int:
        f = self._b.lib.ref_rng_next_u64 if self._b.is_ref else self._b.lib.orc_rng_next_u64
        return int(f(self.handle))

    def next_below(self, n: int) -> int:
        f = self._b.lib.ref_rng_next_below if self._b.is_ref else self._b.lib.orc_rng_next_below
        return int(f(self.handle, C.c_uint64(n)))

    def next_unit(self) -> float:
        f = self._b.lib.ref_rng_next_unit if self._b.is_ref else self._b.lib.orc_rng_next_unit
        return float(f(self.handle))

    def next_gaussian(self, mean: float = 0.0, sd: float = 1.0) -> float:
        f = self._b.lib.ref_rng_next_gaussian if self._b.is_ref else self._b.lib.orc_rng_next_gaussian
        return float(f(self.handle, C.c_double(mean), C.c_double(sd)))

    def gaussian_f32(self, n: int, mean: float = 0.0, sd: float = 1.0) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        if self._b.is_ref:
            for i in range(n):
                out[i] = self.next_gaussian(mean, sd)
        else:
            self._b.lib.orc_rng_fill_gaussian_f32(self.handle, _p(out, _f32p), C.c_int64(n),
                                                  C.c_double(mean), C.c_double(sd))
        return out


class Backend:
    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.is_ref = prefix == "ref_"
        L = self.lib
        if self.is_ref:
            L.ref_rng_new.restype = C.c_void_p
            L.ref_rng_free.argtypes = [C.c_void_p]
            for n in ("ref_rng_next_u64", "ref_rng_next_below"):
                getattr(L, n).restype = C.c_uint64
            L.ref_rng_next_u64.argtypes = [C.c_void_p]
            L.ref_rng_next_below.argtypes = [C.c_void_p, C.c_uint64]
            L.ref_rng_next_unit.restype = C.c_double
            L.ref_rng_next_unit.argtypes = [C.c_void_p]
            L.ref_rng_next_gaussian.restype = C.c_double
            L.ref_rng_next_gaussian.argtypes = [C.c_void_p, C.c_double, C.c_double]
            L.ref_random_subset.restype = C.c_int64
            L.ref_last_error.restype = C.c_char_p
        else:
            L.orc_rng_next_u64.restype = C.c_uint64
            L.orc_rng_next_below.restype = C.c_uint64
            L.orc_rng_next_unit.restype = C.c_double
            L.orc_rng_next_gaussian.restype = C.c_double
            L.orc_random_subset.restype = C.c_int64

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, st: int, where: str):
        if st != 0:
            raise OracleError(st, where)

    def rng(self, seed: int) -> Rng:
        return Rng(self, seed)

    # ---- synapse.cpp ---------------------------------------------------
    def softmax(self, scores) -> np.ndarray:
        s = _f64(scores)
        out = np.empty_like(s)
        self._check(self._fn("softmax")(_p(s, _f64p), C.c_int64(s.size), _p(out, _f64p)), "softmax")
        return out

    def argmax(self, v) -> int:
        vv = _f32(v).reshape(-1)
        if self.is_ref:
            out = C.c_int()
            self._check(self.lib.ref_argmax(_p(vv, _f32p), C.c_int64(vv.size), C.byref(out)), "argmax")
            return int(out.value)
        return int(self.lib.orc_argmax(_p(vv, _f32p), C.c_int64(vv.size)))

    def attention_scores_points(self, keys, query, n_heads: int) -> np.ndarray:
        k = _f32(keys)
        count, dim = (k.shape[0], k.shape[1]) if k.ndim == 2 else (0, int(k.shape[-1]) if k.ndim else 0)
        q = _f32(query)
        out = np.empty(count, dtype=np.float64)
        st = self._fn("attention_scores_points")(_p(k, _f32p), C.c_int64(count), C.c_int(dim), _p(q, _f32p),
                                                 C.c_int64(q.size), C.c_int(n_heads), _p(out, _f64p))
        self._check(st, "attention_scores_points")
        return out

    def coverage_scores_points(self, cloud, selected=()) -> np.ndarray:
        c = _f32(cloud)
        s = _i64(np.asarray(selected, dtype=np.int64).reshape(-1))
        out = np.empty(c.shape[0], dtype=np.float64)
        st = self._fn("coverage_scores_points")(_p(c, _f32p), C.c_int64(c.shape[0]), C.c_int(c.shape[1]),
                                                _p(s, _i64p), C.c_int64(s.size), _p(out, _f64p))
        self._check(st, "coverage_scores_points")
        return out

    def select_landmarks_points(self, cloud, attention, k: int, lam: float):
        c = _f32(cloud)
        a = _f64(attention)
        cap = max(1, min(max(k, 0), c.shape[0]))
        idx = np.empty(cap, dtype=np.int64)
        sc = np.empty(cap, dtype=np.float64)
        n = C.c_int64(0)
        st = self._fn("select_landmarks_points")(_p(c, _f32p), C.c_int64(c.shape[0]), C.c_int(c.shape[1]),
                                                 _p(a, _f64p), C.c_int64(a.size), C.c_int(k), C.c_double(lam),
                                                 _p(idx, _i64p), _p(sc, _f64p), C.byref(n))
        self._check(st, "select_landmarks_points")
        return idx[: n.value].copy(), sc[: n.value].copy()

    # ---- gate.cpp ------------------------------------------------------
    def gate_score(self, h_main, t_side) -> float:
        h, t = _f32(h_main).reshape(-1), _f32(t_side).reshape(-1)
        out = C.c_double(0.0)
        self._check(self._fn("gate_score")(_p(h, _f32p), _p(t, _f32p), C.c_int64(h.size), C.byref(out)), "gate_score")
        return out.value

    def hausdorff_distance(self, cloud, landmarks) -> float:
        c, l = _f32(cloud), _f32(landmarks)
        out = C.c_double(0)
        st = self._fn("hausdorff_distance")(_p(c, _f32p), C.c_int64(c.shape[0]), C.c_int(c.shape[1]),
                                            _p(l, _f32p), C.c_int64(l.shape[0]), C.c_int(l.shape[1]), C.byref(out))
        self._check(st, "hausdorff_distance")
        return out.value

    def hausdorff_to_subset(self, cloud, rows) -> float:
        c, r = _f32(cloud), _i64(rows)
        out = C.c_double(0)
        st = self._fn("hausdorff_to_subset")(_p(c, _f32p), C.c_int64(c.shape[0]), C.c_int(c.shape[1]),
                                             _p(r, _i64p), C.c_int64(r.size), C.byref(out))
        self._check(st, "hausdorff_to_subset")
        return out.value

    def mean_pairwise_reduction(self, cloud, landmarks) -> float:
        c, l = _f32(cloud), _f32(landmarks)
        out = C.c_double(0)
        st = self._fn("mean_pairwise_reduction")(_p(c, _f32p), C.c_int64(c.shape[0]), C.c_int(c.shape[1]),
                                                 _p(l, _f32p), C.c_int64(l.shape[0]), C.c_int(l.shape[1]),
                                                 C.byref(out))
        self._check(st, "mean_pairwise_reduction")
        return out.value

    def mean_pairwise_reduction_subset(self, cloud, rows) -> float:
        c, r = _f32(cloud), _i64(rows)
        out = C.c_double(0)
        st = self._fn("mean_pairwise_reduction_subset")(_p(c, _f32p), C.c_int64(c.shape[0]), C.c_int(c.shape[1]),
                                                        _p(r, _i64p), C.c_int64(r.size), C.byref(out))
        self._check(st, "mean_pairwise_reduction_subset")
        return out.value

    # ---- kernels.cpp ---------------------------------------------------
    def attend(self, q, keys, values, n_entries: int, n_heads: int, d_k: int) -> np.ndarray:
        qq, kk, vv = _f32(q), _f32(keys), _f32(values)
        out = np.empty(n_heads * d_k, dtype=np.float32)
        f = self._fn("attend")
        if self.is_ref:
            self._check(f(_p(qq, _f32p), _p(kk, _f32p), _p(vv, _f32p), C.c_int64(n_entries), C.c_int(n_heads),
                          C.c_int(d_k), _p(out, _f32p)), "attend")
        else:
            f(_p(qq, _f32p), _p(kk, _f32p), _p(vv, _f32p), C.c_int64(n_entries), C.c_int(n_heads), C.c_int(d_k),
              _p(out, _f32p))
        return out

    def decode_attend(self, syn_k, syn_v, tail_k, tail_v, tail_len, q, n_threads: int | None = None) -> np.ndarray:
        """Expected batched-decode outputs: attend (n_heads = 1) per (agent, layer,
        q-head) over [synapse rows || private rows [0, tail_len[a])]
        (orc_decode_attend_agents).  Agents are split over host threads: the C
        call releases the GIL."""
        import threading
        if self.is_ref:
            raise NotImplementedError("decode_attend is a restatement-side composition")
        sk, sv, tk, tv, qq = _f32(syn_k), _f32(syn_v), _f32(tail_k), _f32(tail_v), _f32(q)
        tl = np.ascontiguousarray(tail_len, dtype=np.int32)
        n, n_layers, n_q, d_k = qq.shape
        n_kv, k_syn, t_cap = sk.shape[1], sk.shape[2], tk.shape[3]
        out = np.empty_like(qq)
        f = self._fn("decode_attend_agents")
        n_threads = max(1, min(n, n_threads or (os.cpu_count() or 1)))

        def run(a0, a1):
            f(C.c_int64(a0), C.c_int64(a1), n_layers, n_kv, n_q, d_k, C.c_int64(k_syn), C.c_int64(t_cap),
              _p(sk, _f32p), _p(sv, _f32p), _p(tk, _f32p), _p(tv, _f32p), _p(tl, _i32p), _p(qq, _f32p), _p(out, _f32p))

        bounds = [n * i // n_threads for i in range(n_threads + 1)]
        ts = [threading.Thread(target=run, args=(bounds[i], bounds[i + 1])) for i in range(n_threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return out

    # ---- harness/bench.cpp ---------------------------------------------
    def make_clustered_cloud(self, rng: Rng, count: int, dim: int, n_clusters: int, separation: float,
                             sigma: float, rare: int = 4):
        cloud = np.empty((count, dim), dtype=np.float32)
        query = np.empty(dim, dtype=np.float32)
        cl = np.empty(count, dtype=np.int32)
        self._fn("make_clustered_cloud")(rng.handle, C.c_int64(count), C.c_int(dim), C.c_int(n_clusters),
                                         C.c_double(separation), C.c_double(sigma), C.c_int(rare),
                                         _p(cloud, _f32p), _p(query, _f32p), _p(cl, _i32p))
        return cloud, query, cl

    def random_subset(self, rng: Rng, n: int, k: int) -> np.ndarray:
        out = np.empty(max(1, min(n, k)), dtype=np.int64)
        m = self._fn("random_subset")(rng.handle, C.c_int64(n), C.c_int(k), _p(out, _i64p))
        return out[:m].copy()


_ORACLE = None
_REF = None


def build(ref: bool = False) -> None:
    """Run oracle/Makefile (the C restatement; +the reference build if ref)."""
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def load() -> Backend:
    global _ORACLE
    if _ORACLE is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _ORACLE = Backend(ORACLE_SO, "orc_")
    return _ORACLE


def load_ref():
    """The reference library built from /root/reference sources, or None."""
    global _REF
    if _REF is None and os.path.exists(REF_SO):
        _REF = Backend(REF_SO, "ref_")
        _REF.lib.ref_compress_groups_mt.restype = C.c_int
        _REF.lib.ref_decode_attend_mt.restype = C.c_int
    return _REF


def group_attention(backend: Backend, cloud, queries) -> np.ndarray:
    """SURVEY.md §8(d) per-(layer, KV-head) attention: sum, in q-head order, of
    attention_scores_points(cloud, q_h, 1) (composition of synapse.cpp:63-93)."""
    total = np.zeros(np.asarray(cloud).shape[0], dtype=np.float64)
    for q in np.asarray(queries, dtype=np.float32).reshape(-1, np.asarray(cloud).shape[1]):
        total = total + backend.attention_scores_points(cloud, q, 1)
    return total


def synthetic_group(backend: Backend, seed: int, L: int, dim: int, n_q: int):
    """Deterministic synthetic (keys, values, queries) for one selection group,
    drawn from cortex::Rng(seed) in the order keys, values, queries
    (N(0,1) fp32 from cortex::Rng, identical bits host/GPU)."""
    r = backend.rng(seed)
    keys = r.gaussian_f32(L * dim).reshape(L, dim)
    values = r.gaussian_f32(L * dim).reshape(L, dim)
    queries = r.gaussian_f32(n_q * dim).reshape(n_q, dim)
    return keys, values, queries
