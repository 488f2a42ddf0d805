"""cortex:: Referential Injection on the path (proj/include/cortex/injector.hpp):
KvBlock, InjectionRecord, inject() and VirtualPositionPlanner.  The append
itself is an sm_100a kernel on the cache's stream (cx_inject_*).
``encode_thought`` (a full forward pass, injector.cpp:36-68) is out of scope
(SURVEY.md §8(f) "next").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import errors
from ._lib import CxInjectionRecord, c_f32p, check, lib, ptr
from .model import KvCache


@dataclass
class KvBlock:
    """injector.hpp:13-25.  keys/values layout [layer][token][d_model]."""
    base_position: int = 0
    token_count: int = 0
    n_layers: int = 0
    d_model: int = 0
    keys: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    last_hidden: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def key(self, layer: int, t: int) -> np.ndarray:
        d = self.d_model
        o = (layer * self.token_count + t) * d
        return np.asarray(self.keys, np.float32).reshape(-1)[o:o + d]

    def value(self, layer: int, t: int) -> np.ndarray:
        d = self.d_model
        o = (layer * self.token_count + t) * d
        return np.asarray(self.values, np.float32).reshape(-1)[o:o + d]


@dataclass
class InjectionRecord:
    """injector.hpp:27-35."""
    thought_id: int = -1
    token_count: int = 0
    virtual_position_base: int = 0
    applied_at_stream_position: int = 0

    @staticmethod
    def csv_header() -> str:
        return "thought_id,token_count,virtual_position_base,applied_at_stream_position"

    def csv_row(self) -> str:
        return f"{self.thought_id},{self.token_count},{self.virtual_position_base},{self.applied_at_stream_position}"


def inject(river_cache: KvCache, block: KvBlock, thought_id: int, stream_position: int) -> InjectionRecord:
    """injector.hpp:46-47 / injector.cpp:70-94."""
    n = block.n_layers * block.token_count * block.d_model
    k = np.ascontiguousarray(block.keys, np.float32).reshape(-1)
    v = np.ascontiguousarray(block.values, np.float32).reshape(-1)
    if block.token_count >= 1 and (k.size < n or v.size < n):
        raise errors.precondition_error("inject: block arrays shorter than n_layers*token_count*d_model")
    rec = CxInjectionRecord()
    check(lib.cx_inject_host(river_cache.handle, ptr(k, c_f32p) if k.size else None,
                             ptr(v, c_f32p) if v.size else None, int(block.base_position), int(block.token_count),
                             int(block.n_layers), int(block.d_model), int(thought_id), int(stream_position),
                             C.byref(rec)), "inject")
    return InjectionRecord(rec.thought_id, rec.token_count, rec.virtual_position_base, rec.applied_at_stream_position)


def inject_dev(river_cache: KvCache, keys_dev: int, values_dev: int, base_position: int, token_count: int,
               n_layers: int, d_model: int, thought_id: int, stream_position: int, stream: int = 0) -> InjectionRecord:
    """Device-pointer variant: the block already lives in HBM (e.g. produced by
    a stream agent on the same GPU); the append is stream-ordered."""
    rec = CxInjectionRecord()
    check(lib.cx_inject_dev(river_cache.handle, keys_dev, values_dev, int(base_position), int(token_count),
                            int(n_layers), int(d_model), int(thought_id), int(stream_position), C.byref(rec),
                            stream or None), "inject_dev")
    return InjectionRecord(rec.thought_id, rec.token_count, rec.virtual_position_base, rec.applied_at_stream_position)


class VirtualPositionPlanner:
    """injector.hpp:51-64 / injector.cpp:96-110 (host bookkeeping)."""

    def __init__(self, reserved_start: int, max_positions: int):
        if reserved_start < 0 or reserved_start >= max_positions:
            raise errors.config_error("planner: reserved_start out of range")
        self._start = int(reserved_start)
        self._max = int(max_positions)
        self._used = 0

    def reserved_start(self) -> int:
        return self._start

    def reserve(self, token_count: int) -> int:
        if token_count < 1:
            raise errors.precondition_error("planner: token_count must be >= 1")
        base = self._start + self._used
        if base + token_count > self._max:
            raise errors.capacity_error("planner: reserved virtual range exhausted")
        self._used += token_count
        return base
