"""The B200 batched path on device tensors (torch is plumbing only: device
memory, streams).  Each call is one C-ABI entry point (include/cortex_b200.h)
ordered on the current torch CUDA stream.

Layouts (HBM, fp32):
  keys / values      [G][L][d]              G = n_layers * n_kv selection groups
  queries            [G][P][d_k]            P q-heads per KV head (GQA) or MHA heads
  synapse K / V      [G][take][d]           ascending source rows
  decode tails       [N][n_layers][n_kv][t_cap][d_k]
  decode q / out     [N][n_layers][n_q][d_k]
"""
from __future__ import annotations

import ctypes as C
import threading

import torch

from ._lib import CxDecodeBatch, CxGroups, c_vp, check, lib

SELECT_EXACT_ONLY = 1

_ctx_lock = threading.Lock()
_ctxs = {}


def ctx(device: int | None = None) -> int:
    """Per-(thread, device) cx_ctx (workspace arena)."""
    if device is None:
        device = torch.cuda.current_device()
    key = (threading.get_ident(), device)
    with _ctx_lock:
        h = _ctxs.get(key)
        if h is None:
            p = c_vp()
            check(lib.cx_ctx_create(int(device), C.byref(p)), "ctx_create")
            h = _ctxs[key] = p.value
    return h


LANE_RIVER, LANE_STREAM = 0, 1
_lanes = {}


def lane_stream(lane: str, device: int | None = None) -> torch.cuda.ExternalStream:
    """The context's priority lane as a torch stream: "river" (highest priority:
    injection appends, synapse pushes) or "stream" (medium: agent decode).
    The reference runs these as a river thread and per-agent std::threads
    (scheduler.cpp:63-113, 198); here they are CUDA stream priorities."""
    if device is None:
        device = torch.cuda.current_device()
    code = {"river": LANE_RIVER, "stream": LANE_STREAM}[lane]
    key = (threading.get_ident(), device, code)
    s = _lanes.get(key)
    if s is None:
        p, prio = c_vp(), C.c_int()
        check(lib.cx_ctx_lane_stream(ctx(device), code, C.byref(p), C.byref(prio)), "ctx_lane_stream")
        s = _lanes[key] = torch.cuda.ExternalStream(p.value, device=torch.device("cuda", device))
        s.cx_priority = prio.value
    return s


class _DevView:
    """__cuda_array_interface__ over memory owned by the library (zero copy)."""

    def __init__(self, ptr: int, shape, strides_elems, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "strides": tuple(4 * s for s in strides_elems), "version": 3}
        self._owner = owner


def kvcache_head_view(cache, kv_head: int, count: int | None = None, values: bool = False) -> torch.Tensor:
    """Zero-copy [n_layers, count, d_k] view of one KV head of a device KvCache
    (layout [layer][capacity][d_model], model.hpp:100-103): the per-(layer, KV
    head) selection groups of the river's context rows (count defaults to the
    cache size)."""
    cfg = cache.config()
    cap = cache.capacity()
    n = cache.size() if count is None else int(count)
    base = cache.values_dev() if values else cache.keys_dev()
    v = _DevView(base + 4 * kv_head * cfg.d_k, (cfg.n_layers, n, cfg.d_k), (cap * cfg.d_model, cfg.d_model, 1), cache)
    return torch.as_tensor(v, device=torch.device("cuda", torch.cuda.current_device()))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _groups(keys: torch.Tensor, queries: torch.Tensor | None, mode: str) -> CxGroups:
    if keys.dtype != torch.float32 or not keys.is_cuda:
        raise TypeError("keys must be a CUDA float32 tensor [G, L, d]")
    G, L, d = keys.shape
    if keys.stride(2) != 1:
        raise ValueError("keys rows must be contiguous")
    g = CxGroups()
    g.n_groups, g.count, g.dim = G, L, d
    g.clouds = keys.data_ptr()
    g.group_stride, g.row_stride = keys.stride(0), keys.stride(1)
    if queries is not None:
        if queries.dtype != torch.float32 or not queries.is_contiguous() or queries.shape[0] != G:
            raise TypeError("queries must be a contiguous CUDA float32 tensor [G, P, d_k]")
        g.queries = queries.data_ptr()
        g.n_pass, g.d_k = queries.shape[1], queries.shape[2]
        g.col_step = g.d_k if mode == "mha" else 0
    return g


def attention_grouped(keys: torch.Tensor, queries: torch.Tensor, mode: str = "gqa") -> torch.Tensor:
    """Attention mass per row of every group -> [G, L] fp64 (synapse.cpp:63-93)."""
    g = _groups(keys, queries, mode)
    out = torch.empty((g.n_groups, g.count), dtype=torch.float64, device=keys.device)
    check(lib.cx_attention_grouped_dev(ctx(keys.device.index), C.byref(g), out.data_ptr(), _stream()),
          "attention_grouped")
    return out


def select_grouped(keys: torch.Tensor, attention: torch.Tensor, k: int, lam: float, flags: int = 0):
    """Greedy hybrid selection per group -> (rows [G, take] int64, scores [G, take] fp64)."""
    g = _groups(keys, None, "gqa")
    take = min(k, g.count)
    rows = torch.empty((g.n_groups, max(take, 0)), dtype=torch.int64, device=keys.device)
    scores = torch.empty((g.n_groups, max(take, 0)), dtype=torch.float64, device=keys.device)
    att = attention.contiguous()
    check(lib.cx_select_grouped_dev(ctx(keys.device.index), C.byref(g), att.data_ptr(), int(k), float(lam),
                                    int(flags), rows.data_ptr(), scores.data_ptr(), _stream()), "select_grouped")
    return rows, scores


def gather_rows(src: torch.Tensor, rows: torch.Tensor, dst: torch.Tensor) -> torch.Tensor:
    """Landmark gather: dst[g, s] = src[g, rows[g, s]] (synapse.cpp:303-318 copy)."""
    g = _groups(src, None, "gqa")
    if not rows.is_contiguous() or rows.dtype != torch.int64 or not dst.is_contiguous():
        raise TypeError("rows must be contiguous int64 [G, take]; dst contiguous [G, take, d]")
    check(lib.cx_gather_grouped_dev(ctx(src.device.index), C.byref(g), src.data_ptr(), rows.data_ptr(),
                                    int(rows.shape[1]), dst.data_ptr(), _stream()), "gather_rows")
    return dst


def compress_grouped(keys: torch.Tensor, values: torch.Tensor, queries: torch.Tensor, k: int, lam: float,
                     mode: str = "gqa", flags: int = 0, out=None):
    """One synapse compression for G groups: attention + greedy selection +
    landmark K/V gather.  Returns (rows, scores, syn_keys [G,take,d], syn_values)."""
    g = _groups(keys, queries, mode)
    if values.shape != keys.shape or values.stride() != keys.stride():
        raise ValueError("values must match keys' shape and strides")
    take = min(k, g.count)
    if out is None:
        dev = keys.device
        out = (torch.empty((g.n_groups, take), dtype=torch.int64, device=dev),
               torch.empty((g.n_groups, take), dtype=torch.float64, device=dev),
               torch.empty((g.n_groups, take, g.dim), dtype=torch.float32, device=dev),
               torch.empty((g.n_groups, take, g.dim), dtype=torch.float32, device=dev))
    rows, scores, sk, sv = out
    check(lib.cx_compress_grouped_dev(ctx(keys.device.index), C.byref(g), values.data_ptr(), int(k), float(lam),
                                      int(flags), rows.data_ptr(), scores.data_ptr(), sk.data_ptr(), sv.data_ptr(),
                                      _stream()), "compress_grouped")
    return out


def compress_grouped_host(keys: torch.Tensor, values: torch.Tensor, queries: torch.Tensor, k: int, lam: float,
                          mode: str = "gqa", flags: int = 0, out=None, device: int | None = None):
    """The end-to-end compression from HOST tensors (use pinned memory for overlap):
    keys/values [G, L, d], queries [G, P, d_k] (contiguous, CPU) -> host (rows,
    scores, syn_keys, syn_values).  Uploads are chunked and overlap the per-chunk
    compressions inside the library (cx_compress_grouped_host)."""
    for t in (keys, values, queries):
        if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
            raise TypeError("host path: contiguous CPU float32 tensors")
    G, L, d = keys.shape
    if values.shape != keys.shape or queries.shape[0] != G:
        raise ValueError("keys/values/queries shape mismatch")
    P, dk = queries.shape[1], queries.shape[2]
    take = min(k, L)
    if out is None:
        pin = keys.is_pinned()
        out = (torch.empty((G, take), dtype=torch.int64, pin_memory=pin),
               torch.empty((G, take), dtype=torch.float64, pin_memory=pin),
               torch.empty((G, take, d), dtype=torch.float32, pin_memory=pin),
               torch.empty((G, take, d), dtype=torch.float32, pin_memory=pin))
    rows, scores, sk, sv = out
    check(lib.cx_compress_grouped_host(ctx(device), G, L, d, keys.data_ptr(), values.data_ptr(), queries.data_ptr(),
                                       P, dk, dk if mode == "mha" else 0, int(k), float(lam), int(flags),
                                       rows.data_ptr(), scores.data_ptr(), sk.data_ptr(), sv.data_ptr()),
          "compress_grouped_host")
    return out


def decode_step(syn_keys: torch.Tensor, syn_values: torch.Tensor, tail_keys: torch.Tensor,
                tail_values: torch.Tensor, tail_len: torch.Tensor, q: torch.Tensor, out: torch.Tensor,
                new_keys: torch.Tensor | None = None, new_values: torch.Tensor | None = None,
                syn_unchanged: bool = False) -> torch.Tensor:
    """One decode step of N agents against the shared synapse (append + attend).

    syn_*: [n_layers, n_kv, k, d_k]; tail_*: [N, n_layers, n_kv, t_cap, d_k];
    tail_len: [N] int32; q/out: [N, n_layers, n_q, d_k]; new_*: [N, n_layers, n_kv, d_k].
    syn_unchanged: the synapse was not written since the previous step on this stream
    (CX_DECODE_SYN_UNCHANGED: its staging overlaps the previous step's tail).
    """
    n_layers, n_kv, k_syn, d_k = syn_keys.shape
    N, _, _, t_cap, _ = tail_keys.shape
    n_q = q.shape[2]
    for t in (syn_keys, syn_values, tail_keys, tail_values, q, out):
        if not t.is_contiguous() or t.dtype != torch.float32:
            raise TypeError("decode tensors must be contiguous float32")
    if tail_len.dtype != torch.int32:
        raise TypeError("tail_len must be int32")
    b = CxDecodeBatch()
    b.n_agents, b.n_layers, b.n_kv, b.n_q, b.d_k, b.k_syn = N, n_layers, n_kv, n_q, d_k, k_syn
    b.syn_keys, b.syn_values = syn_keys.data_ptr(), syn_values.data_ptr()
    b.tail_keys, b.tail_values = tail_keys.data_ptr(), tail_values.data_ptr()
    b.t_cap = t_cap
    b.tail_len = tail_len.data_ptr()
    b.new_keys = new_keys.data_ptr() if new_keys is not None else None
    b.new_values = new_values.data_ptr() if new_values is not None else None
    b.q, b.out = q.data_ptr(), out.data_ptr()
    b.flags = 1 if syn_unchanged else 0
    check(lib.cx_decode_step_dev(ctx(q.device.index), C.byref(b), _stream()), "decode_step")
    return out


def gate_decide(h: torch.Tensor, t: torch.Tensor, theta: float):
    """gate.cpp:45-61 for every row pair of h / t ([n, dim] float32 CUDA, row-contiguous):
    -> (scores fp64 [n] (NaN when degenerate), accepted bool [n], degenerate bool [n])."""
    if h.shape != t.shape or h.dim() != 2 or h.dtype != torch.float32 or t.dtype != torch.float32:
        raise TypeError("gate_decide: h and t must be float32 [n, dim] of the same shape")
    if h.stride(1) != 1 or t.stride(1) != 1:
        raise ValueError("gate_decide: rows must be contiguous")
    n, dim = h.shape
    scores = torch.empty(n, dtype=torch.float64, device=h.device)
    acc = torch.empty(n, dtype=torch.uint8, device=h.device)
    deg = torch.empty(n, dtype=torch.uint8, device=h.device)
    check(lib.cx_gate_decide_dev(ctx(h.device.index), n, dim, h.data_ptr(), h.stride(0), t.data_ptr(), t.stride(0),
                                 float(theta), scores.data_ptr(), acc.data_ptr(), deg.data_ptr(), _stream()),
          "gate_decide")
    return scores, acc.bool(), deg.bool()


OPTIONS = {"select_cluster": 1, "select_no_sketch": 2, "decode_impl": 3, "decode_ctas_per_lh": 4,
           "host_upload_values": 5, "select_impl": 6, "select_exchange": 7,
           "host_stage_outputs": 8}
DECODE_IMPLS = {"auto": 0, "tc": 1, "v2": 2, "v1": 3}
SELECT_IMPLS = {"auto": 0, "tc": 1, "cuda_core": 2}


def set_option(name: str, value, device: int | None = None) -> int:
    """Path pinning for tests / tuning (cx_ctx_set_option) on this device's ctx;
    returns the previous value.  decode_impl takes "auto" | "tc" | "v2" | "v1"."""
    dev = torch.cuda.current_device() if device is None else device
    code = OPTIONS[name]
    if name == "decode_impl" and isinstance(value, str):
        value = DECODE_IMPLS[value]
    if name == "select_impl" and isinstance(value, str):
        value = SELECT_IMPLS[value]
    old = C.c_int64()
    check(lib.cx_ctx_get_option(ctx(dev), code, C.byref(old)), "ctx_get_option")
    check(lib.cx_ctx_set_option(ctx(dev), code, int(value)), "ctx_set_option")
    return int(old.value)


DEVERR_NONFINITE, DEVERR_TAIL_RANGE = 1, 2


def device_errors(clear: bool = True, device: int | None = None) -> int:
    """Device-detected precondition failures of this device's ctx (cx_ctx_device_errors):
    DEVERR_NONFINITE | DEVERR_TAIL_RANGE bits.  Synchronizes the current stream."""
    dev = torch.cuda.current_device() if device is None else device
    f = C.c_uint()
    check(lib.cx_ctx_device_errors(ctx(dev), _stream(), C.byref(f), int(clear)), "ctx_device_errors")
    return int(f.value)


def selection_gaps(n_groups: int, device: int | None = None) -> torch.Tensor:
    """Decision-gap monitor of the most recent selection on this device's ctx
    (cx_selection_gaps): per group, the smallest top-1 / top-2 exact hybrid gap
    over the greedy rounds, capped at 1e-10; NaN = not monitored."""
    dev = torch.cuda.current_device() if device is None else device
    out = torch.empty(n_groups, dtype=torch.float64, device=torch.device("cuda", dev))
    check(lib.cx_selection_gaps(ctx(dev), int(n_groups), out.data_ptr(), _stream()), "selection_gaps")
    return out


def probe_fp64_rate(device: int | None = None) -> float:
    """Unfused fp64 add / mul operations per second of this device (cx_probe_fp64_rate)."""
    dev = torch.cuda.current_device() if device is None else device
    r = C.c_double()
    check(lib.cx_probe_fp64_rate(ctx(dev), C.byref(r)), "probe_fp64_rate")
    return float(r.value)


def kernel_launch_count() -> int:
    return int(lib.cx_kernel_launch_count())
