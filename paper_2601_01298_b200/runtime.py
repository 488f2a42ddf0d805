"""The River / Stream loop on the device (BASELINE configs[4]):
the device work of Scheduler::run (proj/src/scheduler.cpp:63-113) behind the C-ABI
(cx_cortex_*, csrc/cortex_runtime.cu), plus the device model handles it needs
(Weights, forward_step_dev).

Per river token the library runs, on the context's priority lanes:
  river lane  -- drain_injections (encode_thought + inject, scheduler.cpp:139-156) every
                 ``inject_every`` tokens, the river's forward_step, and a synapse push
                 (scheduler.cpp:158-165) every ``push_every`` tokens into the back buffer;
  stream lane -- every agent x layer decodes one token against the FRONT synapse
                 (a CUDA-graph replay of cx_decode_step_dev).
A push is published (SynapseBuffer::push / read_latest, synapse.hpp:115-135) only once
its completion event has fired; agents never see a partly written synapse.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import device as cxd
from ._lib import CxCortexAgents, CxCortexConfig, CxCortexStats, c_vp, check, lib
from .model import KvCache, ModelConfig


def weights_flat_floats(cfg: ModelConfig) -> int:
    return int(lib.cx_weights_flat_floats(cfg.n_layers, cfg.d_model, cfg.vocab_size))


def random_flat_weights(cfg: ModelConfig, seed: int = 0) -> np.ndarray:
    """A flat weight array in the reference's draw order and distributions
    (model.cpp:49-80: embedding N(0,1), norms N(1,0.02), projections N(0,1/sqrt(d)),
    w_out N(0,1/sqrt(4d))) from numpy's generator -- not WeightStore::init's stream."""
    rng = np.random.default_rng(seed)
    d, dff, v = cfg.d_model, cfg.d_ff(), cfg.vocab_size
    ps, os_ = 1.0 / np.sqrt(d), 1.0 / np.sqrt(dff)
    parts = [rng.normal(0.0, 1.0, v * d)]
    for _ in range(cfg.n_layers):
        parts += [rng.normal(1.0, 0.02, d)] + [rng.normal(0.0, ps, d * d) for _ in range(4)]
        parts += [rng.normal(1.0, 0.02, d), rng.normal(0.0, ps, dff * d), rng.normal(0.0, os_, d * dff)]
    parts += [rng.normal(1.0, 0.02, d), rng.normal(0.0, ps, v * d)]
    flat = np.concatenate(parts).astype(np.float32)
    assert flat.size == weights_flat_floats(cfg)
    return flat


class Weights:
    """Device-resident model weights (cx_weights; WeightStore::device_handle's object)."""

    def __init__(self, cfg: ModelConfig, flat: np.ndarray):
        cfg.validate()
        flat = np.ascontiguousarray(flat, np.float32)
        if flat.size != weights_flat_floats(cfg):
            raise ValueError("flat weights: wrong size for this ModelConfig")
        h = c_vp()
        check(lib.cx_weights_create(cfg.n_layers, cfg.n_heads, cfg.d_model, cfg.d_k, cfg.vocab_size,
                                    cfg.max_positions, cfg.rope_base, flat.ctypes.data, C.byref(h)), "weights_create")
        self._h, self.cfg = h.value, cfg

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.cx_weights_destroy(h)
            self._h = None


def forward_step_dev(weights: Weights, caches, tokens, positions, logits: torch.Tensor | None = None,
                     hidden: torch.Tensor | None = None, final_query: torch.Tensor | None = None) -> None:
    """forward_step (model.cpp:175-235) of len(caches) agents at once on the current
    torch stream: outputs logits [n][vocab], hidden [n][d], final_query [n][d]."""
    n = len(caches)
    hs = (c_vp * n)(*[c.handle for c in caches])
    tk = (C.c_int32 * n)(*[int(t) for t in tokens])
    ps = (C.c_int64 * n)(*[int(p) for p in positions])
    dp = (lambda t: t.data_ptr() if t is not None else None)
    check(lib.cx_forward_step_dev(cxd.ctx(), weights.handle, n, hs, tk, ps, dp(logits), dp(hidden), dp(final_query),
                                  torch.cuda.current_stream().cuda_stream), "forward_step_dev")


class Cortex:
    """One River + N Stream agents on this GPU (cx_cortex).  Tensors (CUDA float32,
    contiguous; kept alive here): tail_keys/values [N][n_layers][n_kv][t_cap][d_k],
    tail_len [N] int32, new_keys/values [N][n_layers][n_kv][d_k], q/out
    [N][n_layers][n_q][d_k], river_queries [n_kv][n_layers][n_q / n_kv][d_k].
    ``river`` holds the prefill (context rows only) and must outlive this object.
    push_mode "scheduler": Scheduler::push_synapse's select_landmarks (last layer, the
    river's final query, scheduler.cpp:158-165); "groups": one selection per (layer, KV
    head) with the fixed ``river_queries`` (the BASELINE cfg2 decomposition)."""

    PUSH_MODES = {"scheduler": 0, "groups": 1}

    def __init__(self, weights: Weights, river: KvCache, *, k: int, lam: float, push_every: int, inject_every: int,
                 thought_tokens: int, virtual_base: int, max_context: int, tail_keys, tail_values, tail_len,
                 new_keys, new_values, q, out, river_queries=None, push_mode: str = "scheduler",
                 gate: bool = False, theta: float = 0.0):
        self._keep = (weights, river, tail_keys, tail_values, tail_len, new_keys, new_values, q, out, river_queries)
        for t in (tail_keys, tail_values, new_keys, new_values, q, out) + ((river_queries,) if river_queries is not None
                                                                          else ()):
            if not t.is_contiguous() or t.dtype != torch.float32 or not t.is_cuda:
                raise TypeError("cortex tensors must be contiguous CUDA float32")
        if tail_len.dtype != torch.int32:
            raise TypeError("tail_len must be int32")
        n, n_layers, n_q, d_k = q.shape
        c = CxCortexConfig(n, n_q, tail_keys.shape[3], int(k), float(lam), int(push_every), int(inject_every),
                           int(thought_tokens), int(virtual_base), int(max_context), self.PUSH_MODES[push_mode],
                           1 if gate else 0, float(theta))
        a = CxCortexAgents(tail_keys.data_ptr(), tail_values.data_ptr(), tail_len.data_ptr(), new_keys.data_ptr(),
                           new_values.data_ptr(), q.data_ptr(), out.data_ptr(),
                           river_queries.data_ptr() if river_queries is not None else None)
        h = c_vp()
        torch.cuda.synchronize()  # the tensors above were produced on torch streams
        check(lib.cx_cortex_create(cxd.ctx(q.device.index), weights.handle, river.handle, C.byref(c), C.byref(a),
                                   C.byref(h)), "cortex_create")
        self._h = h.value
        self.cfg = c
        self.n_layers, self.n_kv, self.d_k = n_layers, river.config().n_heads, d_k
        self.syn_shape = (n_layers, self.n_kv, int(k), d_k)

    def run(self, river_tokens, thought_tokens, agent_steps: int, river_logits: torch.Tensor | None = None,
            synapse_history: torch.Tensor | None = None, out_history: torch.Tensor | None = None):
        """Scheduler::run's device loop: len(river_tokens) river tokens concurrently with
        ``agent_steps`` agent steps.  thought_tokens: ceil(n / inject_every) *
        thought_tokens ids.  Returns (stats dict, the synapse version each agent step
        read).  Audit outputs (optional, device): river_logits [n][vocab],
        synapse_history [V][2][n_layers][n_kv][k][d_k] (indexed by version),
        out_history [agent_steps][N][n_layers][n_q][d_k]."""
        n = len(river_tokens)
        rt = (C.c_int * max(n, 1))(*[int(t) for t in river_tokens])
        tt_list = [int(t) for t in thought_tokens]
        tt = (C.c_int * max(len(tt_list), 1))(*tt_list)
        need = -(-n // self.cfg.inject_every) * self.cfg.thought_tokens
        if len(tt_list) < need:
            raise ValueError(f"cortex.run: {need} thought tokens needed")
        st = CxCortexStats()
        vers = (C.c_uint64 * max(agent_steps, 1))()
        dp = (lambda t: t.data_ptr() if t is not None else None)
        torch.cuda.synchronize()
        check(lib.cx_cortex_run(self._h, n, rt, tt, int(agent_steps), C.byref(st), vers, dp(river_logits),
                                dp(synapse_history),
                                int(synapse_history.shape[0]) if synapse_history is not None else 0,
                                dp(out_history)), "cortex_run")
        stats = {"agent_ms": st.agent_ms, "river_ms": st.river_ms, "push_ms_mean": st.push_ms_mean,
                 "pushes": st.pushes, "injections": st.injections, "last_version": int(st.last_version),
                 "thoughts_accepted": st.thoughts_accepted, "thoughts_rejected": st.thoughts_rejected}
        return stats, np.array(vers[:agent_steps], dtype=np.uint64)

    def gate_log(self):
        """The last run's gate decisions (gate=True): [(thought_id, score, accepted, degenerate)],
        GateDecision's fields (gate.hpp:14-22; score NaN when degenerate)."""
        n = C.c_int64()
        check(lib.cx_cortex_gate_log(self._h, 0, None, None, None, None, C.byref(n)), "cortex_gate_log")
        m = int(n.value)
        ids, sc = (C.c_int64 * max(m, 1))(), (C.c_double * max(m, 1))()
        acc, deg = (C.c_uint8 * max(m, 1))(), (C.c_uint8 * max(m, 1))()
        check(lib.cx_cortex_gate_log(self._h, m, ids, sc, acc, deg, C.byref(n)), "cortex_gate_log")
        return [(int(ids[i]), float(sc[i]), bool(acc[i]), bool(deg[i])) for i in range(m)]

    def front_synapse(self):
        """(keys, values, version) of the latest published synapse."""
        dev = self._keep[2].device
        k = torch.empty(self.syn_shape, dtype=torch.float32, device=dev)
        v = torch.empty_like(k)
        ver = C.c_uint64()
        check(lib.cx_cortex_front_synapse(self._h, k.data_ptr(), v.data_ptr(), C.byref(ver)), "cortex_front_synapse")
        return k, v, int(ver.value)

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            check(lib.cx_cortex_destroy(h), "cortex_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
