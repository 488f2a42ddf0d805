"""cortex:: model-side types on the path: Origin, ModelConfig, KvCache
(proj/include/cortex/model.hpp, config.hpp), backed by the device KvCache of
the C-ABI (cx_kvcache: [n_layers][capacity][d_model] fp32 in HBM).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import errors
from ._lib import c_f32p, c_vp, check, lib, ptr


class Origin(enum.IntEnum):
    """model.hpp:16."""
    context = 0
    injected = 1


@dataclass
class ModelConfig:
    """config.hpp:9-23 (defaults identical)."""
    n_layers: int = 4
    n_heads: int = 4
    d_model: int = 64
    d_k: int = 16
    vocab_size: int = 256
    max_positions: int = 8192
    rope_base: float = 10000.0
    seed: int = 42

    def d_ff(self) -> int:
        return 4 * self.d_model

    def validate(self) -> None:
        """model.cpp:12-21."""
        if self.n_layers < 1 or self.n_heads < 1 or self.d_model < 1 or self.d_k < 1:
            raise errors.config_error("model dimensions must be positive")
        if self.n_heads * self.d_k != self.d_model:
            raise errors.config_error("d_model must equal n_heads * d_k exactly")
        if self.d_k % 2 != 0:
            raise errors.config_error("d_k must be even for pairwise rotation")
        if self.vocab_size < 1:
            raise errors.config_error("vocab_size must be positive")
        if self.max_positions < 1:
            raise errors.config_error("max_positions must be positive")
        if not (self.rope_base > 0.0):
            raise errors.config_error("rope_base must be positive")


class KvCache:
    """model.hpp:67-113 -- per-agent append-only K/V store, device-resident.

    ``key``/``value``/``layer_keys`` read back from HBM (the reference hands out
    spans into host vectors); ``keys_dev``/``values_dev`` give zero-copy device
    pointers for kernels.
    """

    def __init__(self, cfg: ModelConfig, capacity: int = 64):
        cfg.validate()
        self._cfg = cfg
        h = c_vp()
        check(lib.cx_kvcache_create(cfg.n_layers, cfg.n_heads, cfg.d_model, cfg.d_k, cfg.max_positions,
                                    int(capacity), C.byref(h)), "KvCache")
        self._h = h.value

    @property
    def handle(self):
        return self._h

    def config(self) -> ModelConfig:
        return self._cfg

    def size(self) -> int:
        return int(lib.cx_kvcache_size(self._h))

    def positions(self) -> np.ndarray:
        n = self.size()
        p = lib.cx_kvcache_positions_host(self._h)
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.int64)

    def origins(self) -> np.ndarray:
        n = self.size()
        p = lib.cx_kvcache_origins_host(self._h)
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint8)

    def position(self, i: int) -> int:
        return int(self.positions()[i])

    def origin(self, i: int) -> Origin:
        return Origin(int(self.origins()[i]))

    def last_context_position(self) -> int:
        return int(lib.cx_kvcache_last_context_position(self._h))

    def context_count(self) -> int:
        return int(lib.cx_kvcache_context_count(self._h))

    def entry_open(self) -> bool:
        return bool(lib.cx_kvcache_entry_open(self._h))

    def _read(self, layer: int, first: int, n: int):
        d = self._cfg.d_model
        k = np.empty(max(n, 1) * d, np.float32)
        v = np.empty(max(n, 1) * d, np.float32)
        check(lib.cx_kvcache_read(self._h, int(layer), int(first), int(n), ptr(k, c_f32p), ptr(v, c_f32p)),
              "KvCache read")
        return k[: n * d], v[: n * d]

    def key(self, layer: int, i: int) -> np.ndarray:
        return self._read(layer, i, 1)[0]

    def value(self, layer: int, i: int) -> np.ndarray:
        return self._read(layer, i, 1)[1]

    def layer_keys(self, layer: int) -> np.ndarray:
        return self._read(layer, 0, self.size())[0]

    def layer_values(self, layer: int) -> np.ndarray:
        return self._read(layer, 0, self.size())[1]

    @staticmethod
    def entry_bytes(cfg: ModelConfig) -> int:
        return cfg.n_layers * 2 * cfg.d_model * 4

    def kv_bytes(self) -> int:
        return self.size() * self.entry_bytes(self._cfg)

    def begin_entry(self, position: int, origin: Origin) -> None:
        check(lib.cx_kvcache_begin_entry(self._h, int(position), int(origin)), "begin_entry")

    def write_layer(self, layer: int, key, value) -> None:
        k = np.ascontiguousarray(key, np.float32).reshape(-1)
        v = np.ascontiguousarray(value, np.float32).reshape(-1)
        if k.size != v.size:
            raise errors.precondition_error("write_layer: key/value width mismatch")
        check(lib.cx_kvcache_write_layer(self._h, int(layer), ptr(k, c_f32p), ptr(v, c_f32p), k.size), "write_layer")

    def end_entry(self) -> None:
        check(lib.cx_kvcache_end_entry(self._h), "end_entry")

    def append_entry(self, position: int, origin: Origin, keys, values) -> None:
        per = self._cfg.n_layers * self._cfg.d_model
        k = np.ascontiguousarray(keys, np.float32).reshape(-1)
        v = np.ascontiguousarray(values, np.float32).reshape(-1)
        if k.size != per or v.size != per:
            raise errors.precondition_error("append_entry: keys/values must hold n_layers * d_model floats")
        check(lib.cx_kvcache_append_entry(self._h, int(position), int(origin), ptr(k, c_f32p), ptr(v, c_f32p)),
              "append_entry")

    def append_context_dev(self, keys_dev: int, values_dev: int, base_position: int, count: int,
                           stream: int = 0) -> None:
        """Bulk device append of `count` context entries (a river prefill) from a
        device block [n_layers][count][d_model]; same checks as `count`
        append_entry calls (model.cpp:124-173), stream-ordered."""
        check(lib.cx_kvcache_append_context_dev(self._h, keys_dev, values_dev, int(base_position), int(count),
                                                stream or None), "kvcache_append_context_dev")

    def keys_dev(self) -> int:
        return int(lib.cx_kvcache_keys_dev(self._h) or 0)

    def values_dev(self) -> int:
        return int(lib.cx_kvcache_values_dev(self._h) or 0)

    def clone(self) -> "KvCache":
        """A deep copy (KvCache's copy constructor, model.hpp:67-113): rows, positions,
        origins and the append protocol state."""
        h = c_vp()
        check(lib.cx_kvcache_clone(self._h, C.byref(h)), "KvCache clone")
        c = KvCache.__new__(KvCache)
        c._cfg, c._h = self._cfg, h.value
        return c

    def capacity(self) -> int:
        return int(lib.cx_kvcache_capacity(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.cx_kvcache_destroy(h)
            self._h = None
