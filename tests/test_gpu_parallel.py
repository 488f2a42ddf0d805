"""Multi-GPU path with PRODUCT code.

Only one GPU is available here, so ranks that would sit on different GPUs
share cuda:0 and never wait on one another inside a kernel:
* world 2 and 3 over gloo: every rank compresses ITS block of the groups with
  the product kernels, packs its records on the device (cx_synapse_pack_dev),
  ONE all_gather moves them, cx_synapse_unpack_dev lays the synapse out, and
  it equals the single-rank compression of all groups bit for bit;
* the device record exchange emulated at world 2..8 in one process (each
  "rank" compresses its block; the padded blocks are concatenated as an
  all-gather would) -- the unpack's rank-block mapping for even and uneven
  shards;
* the C-ABI NCCL path (cx_comm_init_rank + cx_compress_sharded_dev, whose
  ncclAllGather is the path's one collective) at world 1, bitwise against
  cx_compress_grouped_dev, plus the argument checks of the thought transfer.
"""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

L, D, NQ, K, LAM = 3000, 64, 7, 61, 0.5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(G, seed=5):
    import torch
    gen = torch.Generator(device="cuda").manual_seed(seed)
    kt = torch.randn(G, L, D, device="cuda", generator=gen)
    vt = torch.randn(G, L, D, device="cuda", generator=gen)
    qt = torch.randn(G, NQ, D, device="cuda", generator=gen)
    return kt, vt, qt


def _rank_main(rank, world, port, G, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_01298_b200 import device
        from paper_2601_01298_b200.parallel import all_gather_synapse, shard_range
        kt, vt, qt = _inputs(G)
        b, e = shard_range(G, rank, world)
        part = device.compress_grouped(kt[b:e].contiguous(), vt[b:e].contiguous(), qt[b:e].contiguous(), K, LAM)
        full = all_gather_synapse(*part, G)
        ref = device.compress_grouped(kt, vt, qt, K, LAM)
        torch.cuda.synchronize()
        q.put((rank, all(torch.equal(x, y) for x, y in zip(full, ref))))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,G", [(2, 8), (3, 7)])
def test_sharded_compression_over_gloo_is_bitwise(world, G):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, G, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)], res


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_device_record_exchange_emulated(world):
    import torch

    from paper_2601_01298_b200 import device
    from paper_2601_01298_b200.parallel import pack_synapse, record_bytes, shard_range, unpack_synapse
    G = 11
    kt, vt, qt = _inputs(G, seed=17)
    ref = device.compress_grouped(kt, vt, qt, K, LAM)
    per, rec = -(-G // world), record_bytes(K, D)
    blocks = []
    for r in range(world):
        b, e = shard_range(G, r, world)
        blk = torch.zeros(per * rec, dtype=torch.uint8, device="cuda")
        if e > b:
            part = device.compress_grouped(kt[b:e].contiguous(), vt[b:e].contiguous(), qt[b:e].contiguous(), K, LAM)
            blk[:(e - b) * rec] = pack_synapse(*part, 0, e - b)
        blocks.append(blk)
    full = unpack_synapse(torch.cat(blocks), G, world, K, D)
    torch.cuda.synchronize()
    for x, y in zip(full, ref):
        assert torch.equal(x, y)


def test_nccl_compress_sharded_world1():
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2601_01298_b200 import device, errors
    from paper_2601_01298_b200._lib import lib
    from paper_2601_01298_b200.parallel import Comm
    assert lib.cx_nccl_version() >= 22700
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = Comm.from_torch(device=0)
        rk, nr, dv = C.c_int(), C.c_int(), C.c_int()
        assert lib.cx_comm_info(comm.handle, C.byref(rk), C.byref(nr), C.byref(dv)) == 0
        assert (rk.value, nr.value, dv.value) == (0, 1, 0)
        G = 5
        kt, vt, qt = _inputs(G, seed=23)
        got = comm.compress_sharded(device.ctx(0), kt, vt, qt, K, LAM, G)
        ref = device.compress_grouped(kt, vt, qt, K, LAM)
        torch.cuda.synchronize()
        for x, y in zip(got, ref):
            assert torch.equal(x, y)
        with pytest.raises(errors.precondition_error):  # local groups != this rank's shard
            comm.compress_sharded(device.ctx(0), kt[:3].contiguous(), vt[:3].contiguous(), qt[:3].contiguous(), K,
                                  LAM, G)
        blk = torch.zeros(2, 4, 8, device="cuda")
        with pytest.raises(errors.invalid_argument):  # no other rank to send to
            comm.send_thought(blk, blk, 0)
        comm.close()
    finally:
        dist.destroy_process_group()
