"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): group / agent
sharding and the single synapse all-gather exchange through
the product's host record pack / unpack.  The device path (product selection on
each shard, device pack / unpack, the NCCL communicator) is covered by
tests/test_gpu_parallel.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_01298_b200.parallel import all_gather_synapse, record_bytes, shard_range


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 48, 100, 1000):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_groups, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, e = shard_range(n_groups, rank, world)
        # each rank "selects" its own groups: rows = group id * 1000 + s, K/V encode (g, s)
        take, d = 5, 4
        g = torch.arange(b, e, dtype=torch.int64)[:, None]
        rows = g * 1000 + torch.arange(take)[None]
        scores = rows.to(torch.float64) / 7
        sk = rows[..., None].to(torch.float32).expand(-1, -1, d).contiguous()
        sv = -sk
        full = all_gather_synapse(rows, scores, sk, sv, n_groups)
        exp_rows = torch.arange(n_groups)[:, None] * 1000 + torch.arange(take)[None]
        exp_k = exp_rows[..., None].to(torch.float32).expand(-1, -1, d)
        ok = (torch.equal(full[0], exp_rows) and torch.equal(full[1], exp_rows.to(torch.float64) / 7)
              and torch.equal(full[2], exp_k) and torch.equal(full[3], -exp_k))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_record_layout():
    """cx_synapse_record_bytes: rows + scores + K + V of one group, padded to 256 B."""
    assert record_bytes(164, 64) == ((164 * 16 + 164 * 64 * 8 + 255) // 256) * 256
    assert record_bytes(1, 4) == 256


@pytest.mark.parametrize("n_groups", [48, 7])
def test_all_gather_synapse_world2(n_groups):
    """The exchange step over gloo: the product's host pack / unpack
    (cx_synapse_pack_host / unpack_host) around ONE all_gather."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_groups, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]


def _select_worker(rank, world, port, n_groups, q):
    """Each rank runs the whole greedy selection for its own groups (no
    collective inside selection), then the one all-gather exchange builds the
    full synapse: rows, scores and landmark K/V of every group."""
    import numpy as np

    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = oracle.load()
        b, e = shard_range(n_groups, rank, world)
        L, d, k, lam = 192, 16, 12, 0.5
        rows, scores, sk, sv = [], [], [], []
        for gi in range(b, e):
            keys, values, queries = oracle.synthetic_group(orc, 100 + gi, L, d, 3)
            idx, sc = orc.select_landmarks_points(keys, oracle.group_attention(orc, keys, queries), k, lam)
            rows.append(idx), scores.append(sc), sk.append(keys[idx]), sv.append(values[idx])
        loc = [torch.from_numpy(np.stack(x)) if x else torch.empty((0,) + s)
               for x, s in ((rows, (k,)), (scores, (k,)), (sk, (k, d)), (sv, (k, d)))]
        loc[0] = loc[0].to(torch.int64)
        loc[1] = loc[1].to(torch.float64)
        full = all_gather_synapse(*loc, n_groups)
        ok = True
        for gi in range(n_groups):  # every rank checks every group against a local recompute
            keys, values, queries = oracle.synthetic_group(orc, 100 + gi, L, d, 3)
            idx, sc = orc.select_landmarks_points(keys, oracle.group_attention(orc, keys, queries), k, lam)
            ok &= (np.array_equal(full[0][gi].numpy(), idx) and full[1][gi].numpy().tobytes() == sc.tobytes()
                   and np.array_equal(full[2][gi].numpy(), keys[idx])
                   and np.array_equal(full[3][gi].numpy(), values[idx]))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_groups", [(2, 5), (3, 7)])
def test_sharded_selection_gathers_the_single_rank_synapse(world, n_groups):
    """groups sharded over ranks, one all-gather -> every rank
    holds the synapse a single rank computes, bit for bit (uneven shards)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_select_worker, args=(r, world, port, n_groups, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)]
