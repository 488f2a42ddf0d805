"""River / Stream priority lanes, the bulk river prefill and compression through a
zero-copy KvCache view (cfg5 plumbing, BASELINE configs[4]).

The reference runs the river and each stream agent as std::threads
(scheduler.cpp:63-113, 198); the B200 path runs their device work on CUDA
streams of different priority from one context (SURVEY.md §8(b) threading row).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cx():
    import torch
    torch.cuda.set_device(0)
    import paper_2601_01298_b200 as m
    return m


def test_priority_lanes(cx):
    import torch
    from paper_2601_01298_b200 import device
    river, stream = device.lane_stream("river"), device.lane_stream("stream")
    assert river.cuda_stream != stream.cuda_stream
    # CUDA priorities: numerically smaller = more urgent; the river lane takes the
    # device's greatest priority (torch's own range is a clamped subset of it)
    _, torch_hi = torch.cuda.Stream.priority_range()
    assert river.cx_priority <= torch_hi, "the river lane must have the highest priority"
    assert river.cx_priority < stream.cx_priority <= 0, "stream agents run below the river"
    assert device.lane_stream("river") is river  # one lane object per (thread, device)
    x = torch.ones(1 << 20, device="cuda")
    with torch.cuda.stream(river):
        a = x * 2
    with torch.cuda.stream(stream):
        b = x * 3
    torch.cuda.synchronize()
    assert float(a.sum()) == 2 * (1 << 20) and float(b.sum()) == 3 * (1 << 20)
    with pytest.raises(KeyError):
        device.lane_stream("nope")


def test_append_context_dev(cx):
    """Same checks and partial-append behaviour as repeated append_entry calls
    (model.cpp:124-173)."""
    import torch
    cfg = cx.ModelConfig(n_layers=3, n_heads=2, d_model=8, d_k=4, max_positions=20)
    c = cx.KvCache(cfg, capacity=4)  # grows on the way
    g = torch.Generator(device="cuda").manual_seed(3)
    k = torch.randn(3, 6, 8, device="cuda", generator=g)
    v = torch.randn(3, 6, 8, device="cuda", generator=g)
    c.append_context_dev(k.data_ptr(), v.data_ptr(), 2, 6)
    torch.cuda.synchronize()
    assert c.size() == 6 and c.context_count() == 6 and c.last_context_position() == 7
    assert list(c.positions()) == list(range(2, 8))
    assert all(c.origin(i) == cx.Origin.context for i in range(6))
    for l in range(3):
        assert np.array_equal(c.layer_keys(l).reshape(6, 8), k[l].cpu().numpy())
        assert np.array_equal(c.layer_values(l).reshape(6, 8), v[l].cpu().numpy())
    # non-increasing context position: nothing appended
    with pytest.raises(cx.errors.precondition_error):
        c.append_context_dev(k.data_ptr(), v.data_ptr(), 7, 2)
    assert c.size() == 6
    # runs past max_positions: the entries before the first bad one stay (reference order)
    with pytest.raises(cx.errors.capacity_error):
        c.append_context_dev(k.data_ptr(), v.data_ptr(), 17, 6)
    torch.cuda.synchronize()
    assert c.size() == 9 and list(c.positions()[6:]) == [17, 18, 19]
    assert np.array_equal(c.key(1, 8), k[1, 2].cpu().numpy())
    c2 = cx.KvCache(cfg)
    c2.begin_entry(0, cx.Origin.context)
    with pytest.raises(cx.errors.sequencing_error):
        c2.append_context_dev(k.data_ptr(), v.data_ptr(), 1, 2)
    c.append_context_dev(0, 0, 40, 0)  # empty append is a no-op


def test_compress_through_kvcache_view_and_lanes(cx):
    """A river push: per-KV-head compression of the river cache's context rows
    through the zero-copy [n_layers, L, d_k] view, on the river lane, while an
    injection lands on the same lane -- identical to compressing a contiguous
    copy of the same rows."""
    import torch
    from paper_2601_01298_b200 import device
    from paper_2601_01298_b200.injector import inject_dev
    n_layers, n_kv, dk, L, k = 3, 2, 64, 700, 40
    cfg = cx.ModelConfig(n_layers=n_layers, n_heads=n_kv, d_model=n_kv * dk, d_k=dk, max_positions=4096)
    river = cx.KvCache(cfg, capacity=L + 64)
    g = torch.Generator(device="cuda").manual_seed(9)
    pk = torch.randn(n_layers, L, n_kv * dk, device="cuda", generator=g)
    pv = torch.randn(n_layers, L, n_kv * dk, device="cuda", generator=g)
    rl = device.lane_stream("river")
    with torch.cuda.stream(rl):
        river.append_context_dev(pk.data_ptr(), pv.data_ptr(), 0, L, rl.cuda_stream)
        tk = torch.randn(n_layers, 16, n_kv * dk, device="cuda", generator=g)
        inject_dev(river, tk.data_ptr(), tk.data_ptr(), 2048, 16, n_layers, n_kv * dk, 1, 5, rl.cuda_stream)
        q = torch.randn(n_layers, 7, dk, device="cuda", generator=g)
        res = []
        for h in range(n_kv):
            kh = device.kvcache_head_view(river, h, L)
            vh = device.kvcache_head_view(river, h, L, values=True)
            assert kh.shape == (n_layers, L, dk) and kh.stride() == ((L + 64) * n_kv * dk, n_kv * dk, 1)
            res.append(device.compress_grouped(kh, vh, q, k, 0.5))
    torch.cuda.synchronize()
    assert river.size() == L + 16 and river.context_count() == L
    for h in range(n_kv):
        kc = pk[:, :, h * dk:(h + 1) * dk].contiguous()
        vc = pv[:, :, h * dk:(h + 1) * dk].contiguous()
        rows, scores, sk, sv = device.compress_grouped(kc, vc, q, k, 0.5)
        torch.cuda.synchronize()
        assert torch.equal(rows, res[h][0]) and torch.equal(scores, res[h][1])
        assert torch.equal(sk, res[h][2]) and torch.equal(sv, res[h][3])


@pytest.mark.parametrize("G,pinned,L,k", [(13, True, 1500, 60), (3, False, 1500, 60), (1, True, 700, 30),
                                         (5, True, 40, 64), (48, True, 8192, 164)])
def test_compress_grouped_host_matches_device(cx, G, pinned, L, k):
    """cx_compress_grouped_host (chunked uploads overlapping the per-chunk
    prologues; one selection over all groups when the plan is one wave -- the cfg2 case
    (48, 8192, 164) runs the split plan -- else per-wave selections) ==
    cx_compress_grouped_dev on the same data, bit for bit, including a ragged last chunk
    and pageable host memory."""
    import torch
    from paper_2601_01298_b200 import device
    d, P = 64, 7  # (5, 40, 64): k > L, every row taken (take = min(k, L))
    gen = torch.Generator().manual_seed(21 + G)
    hk = torch.randn(G, L, d, generator=gen)
    hv = torch.randn(G, L, d, generator=gen)
    hq = torch.randn(G, P, d, generator=gen)
    if pinned:
        hk, hv, hq = hk.pin_memory(), hv.pin_memory(), hq.pin_memory()
    rows, scores, sk, sv = device.compress_grouped_host(hk, hv, hq, k, 0.5)
    dr, ds, dsk, dsv = device.compress_grouped(hk.cuda(), hv.cuda(), hq.cuda(), k, 0.5)
    torch.cuda.synchronize()
    assert torch.equal(rows, dr.cpu()) and torch.equal(scores, ds.cpu())
    assert torch.equal(sk, dsk.cpu()) and torch.equal(sv, dsv.cpu())
    with pytest.raises(cx.errors.config_error):
        device.compress_grouped_host(hk, hv, hq, 0, 0.5)


def test_compress_grouped_host_mha_d128(cx):
    """The reference-mode cloud through the host path: a 2-head MHA cache's rows
    (d_model = 128, heads concatenated, col_step = d_k; synapse.cpp:286-320) -- the
    d = 128 selection kernel and the fallback chunking -- == the device path, bitwise."""
    import torch
    from paper_2601_01298_b200 import device
    G, L, dm, H, k = 3, 2100, 128, 2, 45
    gen = torch.Generator().manual_seed(77)
    hk = torch.randn(G, L, dm, generator=gen).pin_memory()
    hv = torch.randn(G, L, dm, generator=gen).pin_memory()
    hq = torch.randn(G, H, dm // H, generator=gen).pin_memory()
    rows, scores, sk, sv = device.compress_grouped_host(hk, hv, hq, k, 0.5, mode="mha")
    dr, ds, dsk, dsv = device.compress_grouped(hk.cuda(), hv.cuda(), hq.cuda(), k, 0.5, mode="mha")
    torch.cuda.synchronize()
    assert torch.equal(rows, dr.cpu()) and torch.equal(scores, ds.cpu())
    assert torch.equal(sk, dsk.cpu()) and torch.equal(sv, dsv.cpu())
    gi = torch.arange(G)[:, None]
    assert torch.equal(sk, hk[gi, rows]) and torch.equal(sv, hv[gi, rows])


def test_append_on_a_caller_stream_orders_before_regrow(cx):
    """An append enqueued on a caller stream behind a long kernel, then a host
    append that regrows the cache (its copies run on the cache's own stream):
    the regrow must wait for the caller-stream append, or its rows are lost."""
    import torch
    cfg = cx.ModelConfig(n_layers=2, n_heads=1, d_model=16, d_k=16, max_positions=64)
    c = cx.KvCache(cfg, capacity=4)
    g = torch.Generator(device="cuda").manual_seed(9)
    k = torch.randn(2, 4, 16, device="cuda", generator=g)
    v = torch.randn(2, 4, 16, device="cuda", generator=g)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)  # ~25 ms: the append below is still queued when the host moves on
        c.append_context_dev(k.data_ptr(), v.data_ptr(), 0, 4, side.cuda_stream)
    nk, nv = np.full(32, 7.0, np.float32), np.full(32, -7.0, np.float32)
    c.append_entry(4, cx.Origin.context, nk, nv)  # capacity 4 -> regrow
    for layer in range(2):
        lk = c.layer_keys(layer).reshape(5, 16)
        assert np.array_equal(lk[:4], k[layer].cpu().numpy()), "rows appended on the caller stream were lost"
        assert np.array_equal(lk[4], nk[16 * layer:16 * layer + 16])
        assert np.array_equal(c.layer_values(layer).reshape(5, 16)[:4], v[layer].cpu().numpy())


@pytest.mark.parametrize("impl", ["tc", "v2", "v1"])
def test_decode_tail_len_out_of_range_is_flagged(cx_option, impl):
    """tail_len == t_cap with an append (no room) and tail_len < 0 raise
    CX_DEVERR_TAIL_RANGE; the offending agents append nothing and no other
    agent's tail changes; a valid batch raises nothing (model.cpp:124-140)."""
    import torch

    from paper_2601_01298_b200 import device
    cx_option("decode_impl", impl)
    N, Lr, H, Q, dk, k, tc = 6, 2, 2, 14, 64, 32, 8
    g = torch.Generator(device="cuda").manual_seed(4)
    sk = torch.randn(Lr, H, k, dk, device="cuda", generator=g)
    sv = torch.randn(Lr, H, k, dk, device="cuda", generator=g)
    tk = torch.randn(N, Lr, H, tc, dk, device="cuda", generator=g)
    tv = torch.randn(N, Lr, H, tc, dk, device="cuda", generator=g)
    nk = torch.randn(N, Lr, H, dk, device="cuda", generator=g)
    nv = torch.randn(N, Lr, H, dk, device="cuda", generator=g)
    q = torch.randn(N, Lr, Q, dk, device="cuda", generator=g)
    out = torch.empty_like(q)
    device.device_errors(clear=True)
    tl = torch.tensor([3, tc - 1, 0, 5, 2, 1], dtype=torch.int32, device="cuda")
    device.decode_step(sk, sv, tk, tv, tl, q, out, nk, nv)
    assert device.device_errors() == 0
    tl_bad = torch.tensor([3, tc, -1, 5, 2, 1], dtype=torch.int32, device="cuda")
    tk0, tv0 = tk.clone(), tv.clone()
    device.decode_step(sk, sv, tk, tv, tl_bad, q, out, nk, nv)
    assert device.device_errors() == device.DEVERR_TAIL_RANGE
    assert torch.equal(tk[1], tk0[1]) and torch.equal(tk[2], tk0[2]), "a flagged agent appended"
    for a in (0, 3, 4, 5):  # the valid agents appended their row and nothing else
        r = int(tl_bad[a])
        assert torch.equal(tk[a][:, :, r], nk[a]) and torch.equal(tv[a][:, :, r], nv[a])
        keep = [i for i in range(tc) if i != r]
        assert torch.equal(tk[a][:, :, keep], tk0[a][:, :, keep])
    device.decode_step(sk, sv, tk, tv, tl, q, out)  # no append: tail_len == t_cap would be valid
    assert device.device_errors() == 0


@pytest.mark.parametrize("G,L,k", [(48, 8192, 164), (13, 1500, 60)])
def test_compress_grouped_host_pinned_outputs(cx, G, L, k):
    """Pinned synapse outputs are written in place by the landmark gather (zero-copy);
    staged (CX_OPT_HOST_STAGE_OUTPUTS = 1) and mixed pinned / pageable outputs take the
    device copy + D2H.  All three give the same bits, equal to the selected host rows."""
    import torch
    from paper_2601_01298_b200 import device
    gen = torch.Generator().manual_seed(5 + G)
    hk = torch.randn(G, L, 64, generator=gen).pin_memory()
    hv = torch.randn(G, L, 64, generator=gen).pin_memory()
    hq = torch.randn(G, 7, 64, generator=gen).pin_memory()

    def outs(pin_k, pin_v):
        return (torch.empty(G, k, dtype=torch.int64).pin_memory(), torch.empty(G, k, dtype=torch.float64).pin_memory(),
                torch.full((G, k, 64), float("nan"), pin_memory=pin_k),
                torch.full((G, k, 64), float("nan"), pin_memory=pin_v))

    zero_copy = device.compress_grouped_host(hk, hv, hq, k, 0.5, out=outs(True, True))
    mixed = device.compress_grouped_host(hk, hv, hq, k, 0.5, out=outs(True, False))
    old = device.set_option("host_stage_outputs", 1)
    try:
        staged = device.compress_grouped_host(hk, hv, hq, k, 0.5, out=outs(True, True))
    finally:
        device.set_option("host_stage_outputs", old)
    for other in (mixed, staged):
        for a, b in zip(zero_copy, other):
            assert torch.equal(a, b)
    gi = torch.arange(G)[:, None]
    rows = zero_copy[0]
    assert torch.equal(zero_copy[2], hk[gi, rows]) and torch.equal(zero_copy[3], hv[gi, rows])
