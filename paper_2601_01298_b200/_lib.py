"""ctypes binding of libcortex_b200.so -- the C-ABI in include/cortex_b200.h.

This is the same binding a maintainer of a Python consumer of the reference
would add.  There is no CPU fallback: if the library is
missing the import fails loudly, and every compute entry point returns
CX_DEVICE_ERROR without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcortex_b200.so")

c_f32p = C.POINTER(C.c_float)
c_f64p = C.POINTER(C.c_double)
c_i64p = C.POINTER(C.c_int64)
c_i32p = C.POINTER(C.c_int32)
c_u8p = C.POINTER(C.c_uint8)
c_vp = C.c_void_p


class CxGroups(C.Structure):
    _fields_ = [
        ("n_groups", C.c_int),
        ("count", C.c_int64),
        ("dim", C.c_int),
        ("clouds", c_vp),
        ("group_stride", C.c_int64),
        ("row_stride", C.c_int64),
        ("queries", c_vp),
        ("n_pass", C.c_int),
        ("d_k", C.c_int),
        ("col_step", C.c_int),
    ]


class CxDecodeBatch(C.Structure):
    _fields_ = [
        ("n_agents", C.c_int), ("n_layers", C.c_int), ("n_kv", C.c_int), ("n_q", C.c_int), ("d_k", C.c_int),
        ("k_syn", C.c_int),
        ("syn_keys", c_vp), ("syn_values", c_vp),
        ("tail_keys", c_vp), ("tail_values", c_vp),
        ("t_cap", C.c_int),
        ("tail_len", c_vp),
        ("new_keys", c_vp), ("new_values", c_vp),
        ("q", c_vp), ("out", c_vp),
        ("flags", C.c_uint),
    ]


class CxInjectionRecord(C.Structure):
    _fields_ = [
        ("thought_id", C.c_int64),
        ("token_count", C.c_int64),
        ("virtual_position_base", C.c_int64),
        ("applied_at_stream_position", C.c_int64),
    ]


class CxCortexConfig(C.Structure):
    _fields_ = [("n_agents", C.c_int), ("n_q", C.c_int), ("t_cap", C.c_int), ("k", C.c_int),
                ("lambda_", C.c_double), ("push_every", C.c_int), ("inject_every", C.c_int),
                ("thought_tokens", C.c_int), ("virtual_base", C.c_int64), ("max_context", C.c_int64),
                ("push_mode", C.c_int), ("gate", C.c_int), ("theta", C.c_double)]


class CxCortexAgents(C.Structure):
    _fields_ = [("tail_keys", c_vp), ("tail_values", c_vp), ("tail_len", c_vp), ("new_keys", c_vp),
                ("new_values", c_vp), ("q", c_vp), ("out", c_vp), ("river_queries", c_vp)]


class CxCortexStats(C.Structure):
    _fields_ = [("agent_ms", C.c_double), ("river_ms", C.c_double), ("push_ms_mean", C.c_double),
                ("pushes", C.c_int), ("injections", C.c_int), ("last_version", C.c_uint64),
                ("thoughts_accepted", C.c_int), ("thoughts_rejected", C.c_int)]


# (name, restype, argtypes); cx_status-returning calls use C.c_int.
_SIGS = [
    ("cx_abi_version", C.c_int, []),
    ("cx_last_error", C.c_char_p, []),
    ("cx_kernel_launch_count", C.c_uint64, []),
    ("cx_attention_scores_points", C.c_int, [c_f32p, C.c_int64, C.c_int, c_f32p, C.c_int64, C.c_int, c_f64p]),
    ("cx_coverage_scores_points", C.c_int, [c_f32p, C.c_int64, C.c_int, c_i64p, C.c_int64, c_f64p]),
    ("cx_select_landmarks_points", C.c_int,
     [c_f32p, C.c_int64, C.c_int, c_f64p, C.c_int64, C.c_int, C.c_double, c_i64p, c_f64p, c_i64p]),
    ("cx_hausdorff_distance", C.c_int, [c_f32p, C.c_int64, C.c_int, c_f32p, C.c_int64, C.c_int, c_f64p]),
    ("cx_hausdorff_to_subset", C.c_int, [c_f32p, C.c_int64, C.c_int, c_i64p, C.c_int64, c_f64p]),
    ("cx_mean_pairwise_reduction", C.c_int, [c_f32p, C.c_int64, C.c_int, c_f32p, C.c_int64, C.c_int, c_f64p]),
    ("cx_mean_pairwise_reduction_subset", C.c_int, [c_f32p, C.c_int64, C.c_int, c_i64p, C.c_int64, c_f64p]),
    ("cx_softmax", C.c_int, [c_f64p, C.c_int64, c_f64p]),
    ("cx_softmax_f32", C.c_int, [c_f32p, C.c_int64, c_f64p]),
    ("cx_argmax", C.c_int, [c_f32p, C.c_int64, C.POINTER(C.c_int)]),
    ("cx_attend", C.c_int, [c_f32p, c_f32p, c_f32p, C.c_int64, C.c_int, C.c_int, c_f32p]),
    ("cx_gate_score", C.c_int, [c_f32p, c_f32p, C.c_int64, c_f64p]),
    ("cx_gate_decide_dev", C.c_int,
     [c_vp, C.c_int64, C.c_int, c_vp, C.c_int64, c_vp, C.c_int64, C.c_double, c_vp, c_vp, c_vp, c_vp]),
    ("cx_ctx_create", C.c_int, [C.c_int, C.POINTER(c_vp)]),
    ("cx_ctx_destroy", C.c_int, [c_vp]),
    ("cx_ctx_lane_stream", C.c_int, [c_vp, C.c_int, C.POINTER(c_vp), C.POINTER(C.c_int)]),
    ("cx_compress_grouped_host", C.c_int,
     [c_vp, C.c_int, C.c_int64, C.c_int, c_vp, c_vp, c_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
      C.c_uint, c_vp, c_vp, c_vp, c_vp]),
    ("cx_attention_grouped_dev", C.c_int, [c_vp, C.POINTER(CxGroups), c_vp, c_vp]),
    ("cx_select_grouped_dev", C.c_int,
     [c_vp, C.POINTER(CxGroups), c_vp, C.c_int, C.c_double, C.c_uint, c_vp, c_vp, c_vp]),
    ("cx_gather_grouped_dev", C.c_int, [c_vp, C.POINTER(CxGroups), c_vp, c_vp, C.c_int, c_vp, c_vp]),
    ("cx_selection_gaps", C.c_int, [c_vp, C.c_int, c_vp, c_vp]),
    ("cx_ctx_set_option", C.c_int, [c_vp, C.c_int, C.c_int64]),
    ("cx_nccl_version", C.c_int, []),
    ("cx_weights_flat_floats", C.c_size_t, [C.c_int, C.c_int, C.c_int]),
    ("cx_weights_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_double, c_vp,
                                     C.POINTER(c_vp)]),
    ("cx_weights_destroy", C.c_int, [c_vp]),
    ("cx_forward_step_dev", C.c_int, [c_vp, c_vp, C.c_int, C.POINTER(c_vp), c_i32p, c_i64p, c_vp, c_vp, c_vp, c_vp]),
    ("cx_device_alloc", C.c_int, [C.c_size_t, C.POINTER(c_vp)]),
    ("cx_device_free", C.c_int, [c_vp]),
    ("cx_device_read", C.c_int, [c_vp, c_vp, C.c_size_t, c_vp]),
    ("cx_matvec", C.c_int, [c_f32p, C.c_int, C.c_int, c_f32p, c_f32p]),
    ("cx_rmsnorm", C.c_int, [c_f32p, c_f32p, C.c_int64, C.c_double, c_f32p]),
    ("cx_elementwise", C.c_int, [c_f32p, c_f32p, C.c_int64, C.c_int]),
    ("cx_apply_rope", C.c_int, [c_f32p, C.c_int64, C.c_int64, C.c_double]),
    ("cx_probe_fp64_rate", C.c_int, [c_vp, C.POINTER(C.c_double)]),
    ("cx_comm_unique_id", C.c_int, [c_vp]),
    ("cx_comm_init_rank", C.c_int, [C.c_int, c_vp, C.c_int, C.c_int, C.POINTER(c_vp)]),
    ("cx_comm_init_all", C.c_int, [C.c_int, c_i32p, C.POINTER(c_vp)]),
    ("cx_comm_destroy", C.c_int, [c_vp]),
    ("cx_comm_info", C.c_int, [c_vp, c_i32p, c_i32p, c_i32p]),
    ("cx_comm_group_start", C.c_int, []),
    ("cx_comm_group_end", C.c_int, []),
    ("cx_compress_sharded_dev", C.c_int,
     [c_vp, c_vp, C.POINTER(CxGroups), c_vp, C.c_int, C.c_int, C.c_double, C.c_uint, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("cx_synapse_record_bytes", C.c_size_t, [C.c_int, C.c_int]),
    ("cx_synapse_pack_dev", C.c_int, [c_vp, c_vp, c_vp, c_vp, C.c_int, C.c_int, C.c_int, C.c_int, c_vp, c_vp]),
    ("cx_synapse_unpack_dev", C.c_int, [c_vp, C.c_int, C.c_int, C.c_int, C.c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("cx_synapse_pack_host", C.c_int, [c_vp, c_vp, c_vp, c_vp, C.c_int, C.c_int, C.c_int, C.c_int, c_vp]),
    ("cx_synapse_unpack_host", C.c_int, [c_vp, C.c_int, C.c_int, C.c_int, C.c_int, c_vp, c_vp, c_vp, c_vp]),
    ("cx_thought_send_dev", C.c_int, [c_vp, c_vp, c_vp, C.c_int64, C.c_int, C.c_int, C.c_int, c_vp]),
    ("cx_thought_recv_dev", C.c_int, [c_vp, c_vp, c_vp, C.c_int64, C.c_int, C.c_int, C.c_int, c_vp]),
    ("cx_ctx_device_errors", C.c_int, [c_vp, c_vp, C.POINTER(C.c_uint), C.c_int]),
    ("cx_ctx_get_option", C.c_int, [c_vp, C.c_int, C.POINTER(C.c_int64)]),
    ("cx_compress_grouped_dev", C.c_int,
     [c_vp, C.POINTER(CxGroups), c_vp, C.c_int, C.c_double, C.c_uint, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("cx_decode_step_dev", C.c_int, [c_vp, C.POINTER(CxDecodeBatch), c_vp]),
    ("cx_compress_grouped_strided_dev", C.c_int,
     [c_vp, C.POINTER(CxGroups), c_vp, C.c_int, C.c_double, C.c_uint, c_vp, c_vp, c_vp, c_vp, C.c_int64, c_vp]),
    ("cx_kvcache_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.POINTER(c_vp)]),
    ("cx_kvcache_destroy", C.c_int, [c_vp]),
    ("cx_kvcache_clone", C.c_int, [c_vp, C.POINTER(c_vp)]),
    ("cx_kvcache_size", C.c_int64, [c_vp]),
    ("cx_kvcache_context_count", C.c_int64, [c_vp]),
    ("cx_kvcache_last_context_position", C.c_int64, [c_vp]),
    ("cx_kvcache_entry_open", C.c_int, [c_vp]),
    ("cx_kvcache_capacity", C.c_int64, [c_vp]),
    ("cx_kvcache_keys_dev", c_vp, [c_vp]),
    ("cx_kvcache_values_dev", c_vp, [c_vp]),
    ("cx_kvcache_positions_host", c_i64p, [c_vp]),
    ("cx_kvcache_origins_host", c_u8p, [c_vp]),
    ("cx_kvcache_begin_entry", C.c_int, [c_vp, C.c_int64, C.c_int]),
    ("cx_kvcache_write_layer", C.c_int, [c_vp, C.c_int, c_f32p, c_f32p, C.c_int64]),
    ("cx_kvcache_end_entry", C.c_int, [c_vp]),
    ("cx_kvcache_append_entry", C.c_int, [c_vp, C.c_int64, C.c_int, c_f32p, c_f32p]),
    ("cx_kvcache_read", C.c_int, [c_vp, C.c_int, C.c_int64, C.c_int64, c_f32p, c_f32p]),
    ("cx_kvcache_append_context_dev", C.c_int, [c_vp, c_vp, c_vp, C.c_int64, C.c_int64, c_vp]),
    ("cx_inject_host", C.c_int,
     [c_vp, c_f32p, c_f32p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64,
      C.POINTER(CxInjectionRecord)]),
    ("cx_inject_dev", C.c_int,
     [c_vp, c_vp, c_vp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64,
      C.POINTER(CxInjectionRecord), c_vp]),
    ("cx_select_landmarks", C.c_int, [c_vp, c_f32p, C.c_int64, C.c_int, C.c_double, C.POINTER(c_vp)]),
    ("cx_snapshot_create", C.c_int,
     [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int64, c_i64p, c_f64p, c_f32p, c_f32p, C.POINTER(c_vp)]),
    ("cx_snapshot_destroy", C.c_int, [c_vp]),
    ("cx_snapshot_release", C.c_int, [c_vp]),
    ("cx_snapshot_version", C.c_uint64, [c_vp]),
    ("cx_snapshot_source_length", C.c_int64, [c_vp]),
    ("cx_snapshot_k_configured", C.c_int, [c_vp]),
    ("cx_snapshot_n_layers", C.c_int, [c_vp]),
    ("cx_snapshot_d_model", C.c_int, [c_vp]),
    ("cx_snapshot_count", C.c_int64, [c_vp]),
    ("cx_snapshot_read", C.c_int, [c_vp, c_i64p, c_f64p, c_f32p, c_f32p]),
    ("cx_snapshot_keys_dev", c_vp, [c_vp]),
    ("cx_snapshot_values_dev", c_vp, [c_vp]),
    ("cx_synapse_buffer_create", C.c_int, [C.POINTER(c_vp)]),
    ("cx_synapse_buffer_destroy", C.c_int, [c_vp]),
    ("cx_synapse_buffer_push", C.c_int, [c_vp, c_vp, C.POINTER(C.c_uint64)]),
    ("cx_synapse_buffer_read_latest", C.c_int, [c_vp, C.POINTER(c_vp)]),
    ("cx_synapse_buffer_wait_nonempty", C.c_int, [c_vp, C.c_int64, C.POINTER(c_vp)]),
    ("cx_synapse_buffer_shutdown", C.c_int, [c_vp]),
    ("cx_cortex_create", C.c_int,
     [c_vp, c_vp, c_vp, C.POINTER(CxCortexConfig), C.POINTER(CxCortexAgents), C.POINTER(c_vp)]),
    ("cx_cortex_run", C.c_int,
     [c_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int, C.POINTER(CxCortexStats),
      C.POINTER(C.c_uint64), c_vp, c_vp, C.c_int, c_vp]),
    ("cx_cortex_front_synapse", C.c_int, [c_vp, c_vp, c_vp, C.POINTER(C.c_uint64)]),
    ("cx_cortex_gate_log", C.c_int, [c_vp, C.c_int64, c_i64p, c_f64p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8),
                                     c_i64p]),
    ("cx_cortex_destroy", C.c_int, [c_vp]),
]

EXPORTED_SYMBOLS = [s[0] for s in _SIGS]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status: int, where: str = "") -> None:
    """Raise the reference-named exception for a non-zero cx_status."""
    if status != 0:
        msg = lib.cx_last_error().decode(errors="replace")
        raise errors.from_status(status, f"{where}: {msg}" if where else msg)


def ptr(a, ct):
    """ctypes pointer to a contiguous numpy array."""
    return a.ctypes.data_as(ct)
