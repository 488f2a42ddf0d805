"""cortex:: synapse API (proj/include/cortex/synapse.hpp) over the B200 C-ABI.

Same names, argument meaning and error types as the reference; every call
runs sm_100a kernels through libcortex_b200.so (include/cortex_b200.h).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import errors
from ._lib import c_f32p, c_f64p, c_i64p, c_vp, check, lib, ptr
from .model import KvCache, Origin


@dataclass
class PointCloud:
    """synapse.hpp:17-26: flat row-major point set."""
    count: int = 0
    dim: int = 0
    data: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    @staticmethod
    def from_rows(rows) -> "PointCloud":
        a = np.ascontiguousarray(rows, dtype=np.float32)
        if a.ndim != 2:
            raise ValueError("rows must be 2-D")
        return PointCloud(a.shape[0], a.shape[1], a.reshape(-1))

    def point(self, i: int) -> np.ndarray:
        return self.data[i * self.dim:(i + 1) * self.dim]


def _cloud(c) -> tuple:
    """(contiguous float32 buffer, count, dim) from a PointCloud or [count, dim] array."""
    if isinstance(c, PointCloud):
        buf = np.ascontiguousarray(c.data, dtype=np.float32).reshape(-1)
        return buf, int(c.count), int(c.dim)
    a = np.ascontiguousarray(c, dtype=np.float32)
    if a.ndim != 2:
        raise ValueError("cloud must be a PointCloud or a 2-D array")
    return a.reshape(-1), a.shape[0], a.shape[1]


@dataclass
class LandmarkEntry:
    """synapse.hpp:30-35."""
    source_position: int
    hybrid_score: float
    keys: np.ndarray    # n_layers * d_model
    values: np.ndarray


class SynapseSnapshot:
    """synapse.hpp:37-49, backed by a device snapshot (cx_snapshot).

    Landmark K/V stay resident in HBM ([n_layers][count][d_model], see
    ``keys_dev``); the host ``landmarks`` list is materialised lazily.
    """

    def __init__(self, handle: Optional[int] = None, *, source_length: int = 0, k_configured: int = 0,
                 n_layers: int = 0, d_model: int = 0, landmarks: Optional[List[LandmarkEntry]] = None):
        self._h = handle
        self._landmarks = landmarks
        self.version = 0
        if handle is None:
            self.source_length, self.k_configured = source_length, k_configured
            self.n_layers, self.d_model = n_layers, d_model
            if self._landmarks is None:
                self._landmarks = []
        else:
            self.source_length = int(lib.cx_snapshot_source_length(handle))
            self.k_configured = int(lib.cx_snapshot_k_configured(handle))
            self.n_layers = int(lib.cx_snapshot_n_layers(handle))
            self.d_model = int(lib.cx_snapshot_d_model(handle))
            self.version = int(lib.cx_snapshot_version(handle))

    @property
    def handle(self):
        return self._h

    @property
    def landmarks(self) -> List[LandmarkEntry]:
        if self._landmarks is None:
            n = int(lib.cx_snapshot_count(self._h))
            per = self.n_layers * self.d_model
            pos = np.empty(max(n, 1), np.int64)
            sc = np.empty(max(n, 1), np.float64)
            ks = np.empty((max(n, 1), per), np.float32)
            vs = np.empty((max(n, 1), per), np.float32)
            check(lib.cx_snapshot_read(self._h, ptr(pos, c_i64p), ptr(sc, c_f64p), ptr(ks, c_f32p), ptr(vs, c_f32p)),
                  "snapshot_read")
            self._landmarks = [LandmarkEntry(int(pos[i]), float(sc[i]), ks[i].copy(), vs[i].copy()) for i in range(n)]
        return self._landmarks

    def kv_bytes(self) -> int:
        return len(self.landmarks) * self.n_layers * 2 * self.d_model * 4

    def to_json(self) -> str:
        """synapse.cpp:322-335 (nlohmann dump: no spaces)."""
        import json
        return json.dumps({"hybrid_scores": [lm.hybrid_score for lm in self.landmarks],
                           "positions": [lm.source_position for lm in self.landmarks],
                           "source_length": self.source_length, "version": self.version},
                          separators=(",", ":"))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None:
            lib.cx_snapshot_release(h)
            self._h = None


def _device_snapshot_from_host(snap: SynapseSnapshot):
    lms = snap.landmarks
    n = len(lms)
    per = snap.n_layers * snap.d_model
    pos = np.ascontiguousarray([lm.source_position for lm in lms] or [0], dtype=np.int64)
    sc = np.ascontiguousarray([lm.hybrid_score for lm in lms] or [0.0], dtype=np.float64)
    if n and per:
        ks = np.ascontiguousarray(np.stack([np.asarray(lm.keys, np.float32).reshape(per) for lm in lms]))
        vs = np.ascontiguousarray(np.stack([np.asarray(lm.values, np.float32).reshape(per) for lm in lms]))
    else:
        ks = vs = np.zeros(1, np.float32)
    h = c_vp()
    check(lib.cx_snapshot_create(snap.source_length, snap.k_configured, snap.n_layers if n else 0,
                                 snap.d_model if n else 0, n if per else 0, ptr(pos, c_i64p), ptr(sc, c_f64p),
                                 ptr(ks, c_f32p), ptr(vs, c_f32p), C.byref(h)), "snapshot_create")
    return h.value


@dataclass
class SelectionResult:
    """synapse.hpp:93-96."""
    indices: np.ndarray
    scores: np.ndarray


@dataclass
class ContextCloud:
    """synapse.hpp:53-57."""
    cloud: PointCloud
    entry_index: np.ndarray
    positions: np.ndarray


def context_key_cloud(cache: KvCache, layer: int) -> ContextCloud:
    """synapse.cpp:48-61: rows with origin == context, in cache order."""
    keys = cache.layer_keys(layer).reshape(cache.size(), cache.config().d_model)
    org = cache.origins()
    idx = np.nonzero(org == int(Origin.context))[0].astype(np.int64)
    rows = keys[idx]
    return ContextCloud(PointCloud(len(idx), cache.config().d_model, rows.reshape(-1).copy()), idx,
                        cache.positions()[idx].copy())


def attention_scores_points(keys, query, n_heads: int) -> np.ndarray:
    """synapse.hpp:62-64."""
    buf, count, dim = _cloud(keys)
    q = np.ascontiguousarray(query, dtype=np.float32).reshape(-1)
    out = np.empty(max(count, 1), np.float64)
    check(lib.cx_attention_scores_points(ptr(buf, c_f32p), count, dim, ptr(q, c_f32p), q.size, n_heads,
                                         ptr(out, c_f64p)), "attention_scores")
    return out[:count]


def attention_scores(cache: KvCache, query, layer: int) -> np.ndarray:
    """synapse.hpp:68-69 / synapse.cpp:95-101."""
    ctx = context_key_cloud(cache, layer)
    if ctx.cloud.count == 0:
        raise errors.precondition_error("attention_scores: cache has no context entries")
    return attention_scores_points(ctx.cloud, query, cache.config().n_heads)


def coverage_scores_points(cloud, selected: Sequence[int] = ()) -> np.ndarray:
    """synapse.hpp:73-74."""
    buf, count, dim = _cloud(cloud)
    sel = np.ascontiguousarray(np.asarray(selected, dtype=np.int64).reshape(-1))
    out = np.empty(max(count, 1), np.float64)
    check(lib.cx_coverage_scores_points(ptr(buf, c_f32p), count, dim, ptr(sel, c_i64p), sel.size,
                                        ptr(out, c_f64p)), "coverage_scores")
    return out[:count] if count else np.zeros(0)


def coverage_scores(cache: KvCache, selected_positions: Sequence[int], layer: int) -> np.ndarray:
    """synapse.hpp:77-79 / synapse.cpp:122-137."""
    ctx = context_key_cloud(cache, layer)
    pos_to_row = {int(p): r for r, p in enumerate(ctx.positions)}
    rows = []
    for p in selected_positions:
        if int(p) not in pos_to_row:
            raise errors.precondition_error("coverage_scores: position is not a context entry")
        rows.append(pos_to_row[int(p)])
    return coverage_scores_points(ctx.cloud, rows)


def hausdorff_distance(cloud, landmarks) -> float:
    """synapse.hpp:83."""
    a, n, d = _cloud(cloud)
    b, m, ld = _cloud(landmarks)
    out = C.c_double(0)
    check(lib.cx_hausdorff_distance(ptr(a, c_f32p), n, d, ptr(b, c_f32p), m, ld, C.byref(out)), "hausdorff_distance")
    return out.value


def hausdorff_to_subset(cloud, landmark_rows: Sequence[int]) -> float:
    """synapse.hpp:84-85."""
    a, n, d = _cloud(cloud)
    r = np.ascontiguousarray(np.asarray(landmark_rows, dtype=np.int64).reshape(-1))
    out = C.c_double(0)
    check(lib.cx_hausdorff_to_subset(ptr(a, c_f32p), n, d, ptr(r, c_i64p), r.size, C.byref(out)), "hausdorff")
    return out.value


def mean_pairwise_reduction(cloud, landmarks) -> float:
    """synapse.hpp:89."""
    a, n, d = _cloud(cloud)
    b, m, ld = _cloud(landmarks)
    out = C.c_double(0)
    check(lib.cx_mean_pairwise_reduction(ptr(a, c_f32p), n, d, ptr(b, c_f32p), m, ld, C.byref(out)),
          "mean_pairwise_reduction")
    return out.value


def mean_pairwise_reduction_subset(cloud, landmark_rows: Sequence[int]) -> float:
    """synapse.hpp:90-91."""
    a, n, d = _cloud(cloud)
    r = np.ascontiguousarray(np.asarray(landmark_rows, dtype=np.int64).reshape(-1))
    out = C.c_double(0)
    check(lib.cx_mean_pairwise_reduction_subset(ptr(a, c_f32p), n, d, ptr(r, c_i64p), r.size, C.byref(out)),
          "mean_pairwise_reduction")
    return out.value


def select_landmarks_points(cloud, attention, k: int, lam: float) -> SelectionResult:
    """synapse.hpp:104-106."""
    buf, count, dim = _cloud(cloud)
    a = np.ascontiguousarray(attention, dtype=np.float64).reshape(-1)
    cap = max(1, min(max(int(k), 0), count))
    idx = np.empty(cap, np.int64)
    sc = np.empty(cap, np.float64)
    n = C.c_int64(0)
    check(lib.cx_select_landmarks_points(ptr(buf, c_f32p), count, dim, ptr(a, c_f64p), a.size, int(k),
                                         float(lam), ptr(idx, c_i64p), ptr(sc, c_f64p), C.byref(n)),
          "select_landmarks")
    return SelectionResult(idx[:n.value].copy(), sc[:n.value].copy())


def select_landmarks(cache: KvCache, query, k: int, lam: float) -> SynapseSnapshot:
    """synapse.hpp:110-111: final-layer context cloud, MHA attention, greedy
    selection, per-layer K/V copy of the winners (all on the device)."""
    q = np.ascontiguousarray(query, dtype=np.float32).reshape(-1)
    h = c_vp()
    check(lib.cx_select_landmarks(cache.handle, ptr(q, c_f32p), q.size, int(k), float(lam), C.byref(h)),
          "select_landmarks")
    return SynapseSnapshot(h.value)


class SynapseBuffer:
    """synapse.hpp:115-135: single-writer multi-reader latest-value buffer."""

    def __init__(self):
        h = c_vp()
        check(lib.cx_synapse_buffer_create(C.byref(h)), "synapse_buffer_create")
        self._h = h.value

    def push(self, snap: SynapseSnapshot) -> int:
        """Stamps and returns the version (1, 2, ...); the buffer takes the
        snapshot over (the reference moves it in, synapse.cpp:337-344)."""
        if snap.handle is None:
            snap._h = _device_snapshot_from_host(snap)
        v = C.c_uint64(0)
        check(lib.cx_synapse_buffer_push(self._h, snap.handle, C.byref(v)), "synapse_buffer_push")
        snap._h = None  # moved-from, like the reference's SynapseSnapshot&&
        return int(v.value)

    def _wrap(self, h) -> Optional[SynapseSnapshot]:
        return None if not h else SynapseSnapshot(h)

    def read_latest(self) -> Optional[SynapseSnapshot]:
        h = c_vp()
        check(lib.cx_synapse_buffer_read_latest(self._h, C.byref(h)), "read_latest")
        return self._wrap(h.value)

    def wait_nonempty(self, timeout_ms: int) -> Optional[SynapseSnapshot]:
        h = c_vp()
        check(lib.cx_synapse_buffer_wait_nonempty(self._h, int(timeout_ms), C.byref(h)), "wait_nonempty")
        return self._wrap(h.value)

    def shutdown(self) -> None:
        check(lib.cx_synapse_buffer_shutdown(self._h), "shutdown")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.cx_synapse_buffer_destroy(h)
            self._h = None
