"""Randomised parity sweeps against the oracle:
* the grouped compression (attention mass -> greedy selection -> landmark K/V
  gather) per group, with seeded random group counts, lengths, k, lambda and widths
  (64: select64, 128: select128, 48 / 96: the generic kernel), clustered and
  duplicated rows, and forced small-cluster row modes -- rows, scores and K/V bit-exact;
* the batched decode on random shapes (ragged tails, q-heads per KV head, append on /
  off) -- within 1e-3, the appended rows bitwise."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    torch.cuda.set_device(0)
    from paper_2601_01298_b200 import device
    return device


@pytest.fixture(scope="module")
def orc():
    return oracle.load()


def _case(seed):
    rs = np.random.default_rng(seed)
    d = int(rs.choice([64, 64, 64, 128, 48, 96]))
    G = int(rs.integers(1, 6))
    L = int(rs.integers(2, 2600))
    k = int(rs.integers(1, min(L, 120) + 1)) if rs.random() < 0.9 else L + 3
    lam = float(rs.choice([0.0, 0.25, 0.5, 0.75, 1.0, rs.random()]))
    nq = int(rs.choice([1, 2, 7]))
    return d, G, L, k, lam, nq


@pytest.mark.parametrize("seed", list(range(24)))
def test_grouped_compress_random_sweep(dev, orc, seed):
    import torch
    d, G, L, k, lam, nq = _case(seed)
    ks, vs, qs = [], [], []
    for gi in range(G):
        keys, values, queries = oracle.synthetic_group(orc, 7000 + 31 * seed + gi, L, d, nq)
        if seed % 3 == 0 and L > 8:  # duplicated rows (exact ties) and a tight cluster
            keys[L // 2] = keys[1]
            keys[: L // 8] = keys[0] + 1e-3 * keys[: L // 8]
        ks.append(keys)
        vs.append(values)
        qs.append(queries)
    kt = torch.from_numpy(np.stack(ks)).cuda()
    vt = torch.from_numpy(np.stack(vs)).cuda()
    qt = torch.from_numpy(np.stack(qs)).cuda()
    rows, scores, sk, sv = dev.compress_grouped(kt, vt, qt, k, lam)
    gaps = dev.selection_gaps(G).cpu().numpy()
    a = dev.attention_grouped(kt, qt)
    torch.cuda.synchronize()
    rows, scores = rows.cpu().numpy(), scores.cpu().numpy()
    sk, sv, a = sk.cpu().numpy(), sv.cpu().numpy(), a.cpu().numpy()
    for gi in range(G):
        idx, sc = orc.select_landmarks_points(ks[gi], a[gi], k, lam)  # the device attention, same input
        assert rows[gi].tobytes() == idx.tobytes(), (seed, gi, d, L, k, lam)
        assert scores[gi].tobytes() == sc.tobytes(), (seed, gi)
        assert np.array_equal(sk[gi], ks[gi][idx]) and np.array_equal(sv[gi], vs[gi][idx])
        # end to end: the oracle's own attention gives the same index set whenever the
        # decision-gap monitor certifies it (every round's top-1 / top-2 gap > 1e-11, far above
        # the attention's last-ulp exp differences), which includes the near-duplicate
        # clusters above; on unmonitored (generic-dim) groups only unperturbed N(0,1) data
        # is checked end to end (its gaps dwarf the exp noise)
        certified = bool(gaps[gi] > 1e-11)
        if certified or (np.isnan(gaps[gi]) and seed % 3 != 0):
            a_ref = oracle.group_attention(orc, ks[gi], qs[gi])
            idx_ref, _ = orc.select_landmarks_points(ks[gi], a_ref, k, lam)
            assert np.array_equal(rows[gi], idx_ref), (seed, gi, float(gaps[gi]))
        elif d in (64, 128):
            # monitored and NOT certified: only exact ties from the duplicated rows may do that
            assert seed % 3 == 0 and gaps[gi] == 0.0, (seed, gi, float(gaps[gi]))


@pytest.mark.parametrize("impl", ["cuda_core", "tc_cluster", "tc_coop", "tc_split"])
@pytest.mark.parametrize("seed", list(range(12)))
def test_grouped_compress_forced_row_modes(dev, orc, cx_option, seed, impl):
    """The same check with the cluster size forced small (CX_OPT_SELECT_CLUSTER): for the CUDA-core
    kernel the rows beyond the register rows live in shared memory as fp32 or as the fp16 sketch;
    for the tensor-core kernel the sketch tiles split between shared memory and TMEM, with the
    exchanges through DSMEM (clusters) or global memory (cooperative launch)."""
    import torch
    if impl == "cuda_core":
        cx_option("select_impl", "cuda_core")
    else:
        cx_option("select_impl", "tc")
        cx_option("select_exchange", {"tc_cluster": 1, "tc_coop": 2, "tc_split": 3}[impl])
    rs = np.random.default_rng(500 + seed)
    d = int(rs.choice([64, 64, 128]))
    C = int(rs.integers(2, 7))
    L = int(rs.integers(2500, 7000)) if d == 64 else int(rs.integers(800, 2000))
    k = int(rs.integers(10, 90))
    lam = float(rs.choice([0.3, 0.5, 0.8]))
    if (L + C - 1) // C > 2048:
        C = (L + 2047) // 2048
    if impl != "cuda_core" and d != 64:
        pytest.skip("the tensor-core selection is d = 64")
    cx_option("select_cluster", C)
    G = 2
    ks, vs, qs = zip(*[oracle.synthetic_group(orc, 9100 + 7 * seed + gi, L, d, 2) for gi in range(G)])
    kt = torch.from_numpy(np.stack(ks)).cuda()
    vt = torch.from_numpy(np.stack(vs)).cuda()
    qt = torch.from_numpy(np.stack(qs)).cuda()
    rows, scores, sk, sv = dev.compress_grouped(kt, vt, qt, k, lam)
    a = dev.attention_grouped(kt, qt)
    torch.cuda.synchronize()
    rows, scores, sk, a = rows.cpu().numpy(), scores.cpu().numpy(), sk.cpu().numpy(), a.cpu().numpy()
    for gi in range(G):
        idx, sc = orc.select_landmarks_points(ks[gi], a[gi], k, lam)
        assert rows[gi].tobytes() == idx.tobytes(), (seed, gi, d, C, L, k)
        assert scores[gi].tobytes() == sc.tobytes(), (seed, gi)
        assert np.array_equal(sk[gi], ks[gi][idx])


@pytest.mark.parametrize("seed", list(range(16)))
def test_decode_random_sweep(dev, orc, seed):
    """Batched decode (default dispatch: tcgen05 -> v2 -> v1) on seeded random shapes:
    agents, synapse size, tail capacity, ragged per-agent tail lengths, q-heads per KV
    head, layers, KV heads, with and without the fused append; every (agent, layer,
    q-head) output within 1e-3 (unit floor) of the oracle's attend over
    [synapse rows || private rows || new row], and the appended row bitwise."""
    import torch
    rs = np.random.default_rng(900 + seed)
    N = int(rs.integers(1, 40))
    Lr = int(rs.integers(1, 3))
    H = int(rs.integers(1, 3))
    qpg = int(rs.choice([1, 2, 4, 7, 8]))
    Q = H * qpg
    dk = 64
    k = int(rs.integers(1, 177))
    Tc = int(rs.integers(1, 65))
    app = bool(rs.random() < 0.8)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    syn_k = torch.randn(Lr, H, k, dk, device="cuda", generator=gen)
    syn_v = torch.randn(Lr, H, k, dk, device="cuda", generator=gen)
    tk = torch.randn(N, Lr, H, Tc, dk, device="cuda", generator=gen)
    tv = torch.randn(N, Lr, H, Tc, dk, device="cuda", generator=gen)
    hi = Tc - 1 if app else Tc
    tl = torch.randint(0, hi + 1, (N,), device="cuda", generator=gen).to(torch.int32)
    nk = torch.randn(N, Lr, H, dk, device="cuda", generator=gen) if app else None
    nv = torch.randn(N, Lr, H, dk, device="cuda", generator=gen) if app else None
    q = torch.randn(N, Lr, Q, dk, device="cuda", generator=gen)
    out = torch.empty_like(q)
    dev.decode_step(syn_k, syn_v, tk, tv, tl, q, out, nk, nv)
    torch.cuda.synchronize()
    o, tkn, tvn, tln = out.cpu().numpy(), tk.cpu().numpy(), tv.cpu().numpy(), tl.cpu().numpy()
    sk, sv, qn = syn_k.cpu().numpy(), syn_v.cpu().numpy(), q.cpu().numpy()
    nkn = nk.cpu().numpy() if app else None
    nvn = nv.cpu().numpy() if app else None
    worst = 0.0
    for a in range(N):
        n_t = int(tln[a]) + (1 if app else 0)
        for l in range(Lr):
            for g in range(H):
                if app:  # the fused append wrote row tail_len
                    assert np.array_equal(tkn[a, l, g, tln[a]], nkn[a, l, g])
                    assert np.array_equal(tvn[a, l, g, tln[a]], nvn[a, l, g])
                kk = np.concatenate([sk[l, g], tkn[a, l, g, :n_t]])
                vv = np.concatenate([sv[l, g], tvn[a, l, g, :n_t]])
                for hh in range(qpg):
                    h = g * qpg + hh
                    exp = orc.attend(qn[a, l, h], kk, vv, k + n_t, 1, dk)
                    worst = max(worst, float(np.max(np.abs(o[a, l, h] - exp) / np.maximum(1.0, np.abs(exp)))))
    assert worst <= 1e-3, (seed, worst, N, k, Tc, qpg)


@pytest.mark.parametrize("N,lo,hi", [(100, 13, 37), (100, 0, 50), (64, 63, 64)])
def test_decode_agent_shard_is_bitwise(dev, N, lo, hi):
    """SURVEY.md §8(e) agent sharding: a rank decodes a contiguous block of
    agents on its own; every agent's output and appended rows must equal, bit
    for bit, the same agent's result inside the full batch (tile membership,
    grid shape and CTA count differ between the two launches)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(N + lo)
    Lr, H, Q, dk, T, k = 3, 2, 14, 64, 33, 164
    syn_k = torch.randn(Lr, H, k, dk, device="cuda", generator=g)
    syn_v = torch.randn(Lr, H, k, dk, device="cuda", generator=g)
    tk = torch.randn(N, Lr, H, T, dk, device="cuda", generator=g)
    tv = torch.randn(N, Lr, H, T, dk, device="cuda", generator=g)
    tl = torch.randint(0, T, (N,), dtype=torch.int32, device="cuda", generator=g)
    nk = torch.randn(N, Lr, H, dk, device="cuda", generator=g)
    nv = torch.randn(N, Lr, H, dk, device="cuda", generator=g)
    q = torch.randn(N, Lr, Q, dk, device="cuda", generator=g)
    tk_s, tv_s = tk[lo:hi].clone(), tv[lo:hi].clone()
    out = torch.empty_like(q)
    dev.decode_step(syn_k, syn_v, tk, tv, tl, q, out, nk, nv)
    out_s = torch.empty_like(q[lo:hi])
    dev.decode_step(syn_k, syn_v, tk_s, tv_s, tl[lo:hi].contiguous(), q[lo:hi].contiguous(), out_s,
                    nk[lo:hi].contiguous(), nv[lo:hi].contiguous())
    torch.cuda.synchronize()
    assert torch.equal(out[lo:hi], out_s)
    assert torch.equal(tk[lo:hi], tk_s) and torch.equal(tv[lo:hi], tv_s)
