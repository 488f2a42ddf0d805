"""Multi-GPU sharding of the hot path.

* Selection groups (layer, KV-head) are independent: rank r owns a contiguous
  block of groups and runs the whole k-round greedy loop locally -- no
  collective during selection.  The single exchange step packs each rank's
  landmark rows / scores / K / V into fixed-size per-group records
  (cx_synapse_pack_dev) and all-gathers them in ONE collective, after which
  cx_synapse_unpack_dev lays out the full synapse on every GPU.
  - `Comm` + `compress_sharded`: the C-ABI path (cx_compress_sharded_dev), one
    NCCL communicator per rank (ncclAllGather over NVLink / NVSwitch);
  - `all_gather_synapse`: the same records over any torch.distributed group
    (gloo in the CPU tests, NCCL otherwise).
* Decode shards by agent: rank r owns a contiguous block of agents and
  attends against its local synapse replica -- no per-step exchange.
* Accepted thoughts from a non-river GPU reach the river GPU with
  `Comm.send_thought` / `Comm.recv_thought` (cx_thought_send_dev / recv_dev).
"""
from __future__ import annotations

import ctypes as C
from typing import Tuple

import torch
import torch.distributed as dist

from ._lib import check, lib


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Balanced contiguous [begin, end) block of n items for `rank` of `world`
    (the first n % world ranks hold one more; comm.cu shard())."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def record_bytes(take: int, dim: int) -> int:
    return int(lib.cx_synapse_record_bytes(int(take), int(dim)))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def pack_synapse(rows, scores, syn_k, syn_v, g_begin: int, n_groups: int) -> torch.Tensor:
    """Groups [g_begin, g_begin + n_groups) of the [G] synapse arrays -> n_groups
    consecutive records (uint8 tensor on the arrays' device; cx_synapse_pack_dev /
    cx_synapse_pack_host)."""
    take, dim = syn_k.shape[1], syn_k.shape[2]
    out = torch.empty(n_groups * record_bytes(take, dim), dtype=torch.uint8, device=syn_k.device)
    args = (rows.data_ptr(), scores.data_ptr(), syn_k.data_ptr(), syn_v.data_ptr(), int(g_begin), int(n_groups), take,
            dim, out.data_ptr())
    if syn_k.is_cuda:
        check(lib.cx_synapse_pack_dev(*args, _stream()), "synapse_pack")
    else:
        check(lib.cx_synapse_pack_host(*args), "synapse_pack")
    return out


def unpack_synapse(records: torch.Tensor, n_groups: int, world: int, take: int, dim: int, out=None):
    """`world` padded blocks of ceil(G / world) records -> (rows, scores, syn_k, syn_v) [G]."""
    dev = records.device
    if out is None:
        out = (torch.empty(n_groups, take, dtype=torch.int64, device=dev),
               torch.empty(n_groups, take, dtype=torch.float64, device=dev),
               torch.empty(n_groups, take, dim, device=dev), torch.empty(n_groups, take, dim, device=dev))
    rows, scores, sk, sv = out
    args = (records.data_ptr(), int(n_groups), int(world), int(take), int(dim), rows.data_ptr(), scores.data_ptr(),
            sk.data_ptr(), sv.data_ptr())
    if records.is_cuda:
        check(lib.cx_synapse_unpack_dev(*args, _stream()), "synapse_unpack")
    else:
        check(lib.cx_synapse_unpack_host(*args), "synapse_unpack")
    return out


def all_gather_synapse(rows, scores, syn_k, syn_v, n_total: int, group=None):
    """This rank's block of groups (shard_range) -> the full synapse on every rank,
    with ONE all_gather of the packed records over a torch.distributed group
    (host or CUDA tensors; with gloo the records travel through host memory).
    Inputs are the local [n_local, ...] tensors; returns [n_total, ...] on their device."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    b, e = shard_range(n_total, rank, world)
    if rows.shape[0] != e - b:
        raise ValueError("local tensors must hold exactly this rank's shard")
    take, dim = syn_k.shape[1], syn_k.shape[2]
    per = -(-n_total // world)
    rec = record_bytes(take, dim)
    send = torch.zeros(per * rec, dtype=torch.uint8, device=syn_k.device)
    if e > b:
        send[:(e - b) * rec] = pack_synapse(rows, scores, syn_k, syn_v, 0, e - b)
    if dist.get_backend(group) == "gloo":
        src = send.cpu()
        bufs = torch.empty(world * per * rec, dtype=torch.uint8)
        dist.all_gather(list(bufs.view(world, per * rec).unbind(0)), src, group=group)
        bufs = bufs.to(syn_k.device)
    else:
        bufs = torch.empty(world * per * rec, dtype=torch.uint8, device=send.device)
        dist.all_gather_into_tensor(bufs, send, group=group)
    return unpack_synapse(bufs, n_total, world, take, dim)


class Comm:
    """One rank of an NCCL communicator owned by the C-ABI (cx_comm).

    `Comm.from_torch()` makes one per rank of the default torch.distributed
    group: rank 0 draws the NCCL unique id and broadcasts it (any backend)."""

    def __init__(self, handle: int, rank: int, world: int, device: int):
        self.handle, self.rank, self.world, self.device = handle, rank, world, device

    @classmethod
    def from_torch(cls, device: int | None = None, group=None) -> "Comm":
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.cuda.current_device() if device is None else device
        uid = (C.c_char * 128)()
        if rank == 0:
            check(lib.cx_comm_unique_id(uid), "comm_unique_id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        check(lib.cx_comm_init_rank(world, uid, rank, dev, C.byref(h)), "comm_init_rank")
        return cls(h.value, rank, world, dev)

    def close(self):
        if self.handle:
            check(lib.cx_comm_destroy(self.handle), "comm_destroy")
            self.handle = None

    def compress_sharded(self, ctx: int, keys, values, queries, k: int, lam: float, n_total: int, out=None,
                         flags: int = 0):
        """cx_compress_sharded_dev: keys/values [n_local, L, d], queries [n_local, P, d] for this
        rank's block of the n_total groups -> the full synapse (rows, scores, syn_k, syn_v) [n_total]."""
        from .device import _groups
        g = _groups(keys, queries, "gqa")
        L, d = keys.shape[1], keys.shape[2]
        take = min(int(k), L)
        dev = keys.device
        if out is None:
            out = (torch.empty(n_total, take, dtype=torch.int64, device=dev),
                   torch.empty(n_total, take, dtype=torch.float64, device=dev),
                   torch.empty(n_total, take, d, device=dev), torch.empty(n_total, take, d, device=dev))
        rows, scores, sk, sv = out
        check(lib.cx_compress_sharded_dev(ctx, self.handle, C.byref(g), values.data_ptr(), int(n_total), int(k),
                                          float(lam), int(flags), rows.data_ptr(), scores.data_ptr(), sk.data_ptr(),
                                          sv.data_ptr(), _stream()), "compress_sharded")
        return out

    def send_thought(self, keys, values, river_rank: int):
        """KvBlock [n_layers, T, d_model] keys / values (CUDA) -> the river GPU."""
        n_layers, T, dm = keys.shape
        check(lib.cx_thought_send_dev(self.handle, keys.data_ptr(), values.data_ptr(), T, n_layers, dm, int(river_rank),
                                      _stream()), "thought_send")

    def recv_thought(self, keys, values, src_rank: int):
        n_layers, T, dm = keys.shape
        check(lib.cx_thought_recv_dev(self.handle, keys.data_ptr(), values.data_ptr(), T, n_layers, dm, int(src_rank),
                                      _stream()), "thought_recv")
