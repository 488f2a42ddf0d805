"""Pin the CPU oracle (oracle/cortex_oracle.c) before trusting it:

1. the reference's own known-answer tests (tests/refcases.py);
2. bit-for-bit agreement with the unmodified reference library built from
   /root/reference sources (oracle/_ref), on randomised inputs -- skipped where
   _ref is not built;
3. the golden fixtures in tests/golden/ (generated from _ref by
   tests/golden/make_golden.py), which travel without /root/reference.
"""
import json
import os

import numpy as np
import pytest

import oracle
import refcases
from conftest import GOLDEN


class OracleApi:
    def __init__(self, b):
        self.b = b

    def __getattr__(self, n):
        return getattr(self.b, n)

    def rng(self, seed):
        return self.b.rng(seed)

    @staticmethod
    def error_kind(e):
        return getattr(e, "kind", type(e).__name__)


@pytest.mark.parametrize("case", refcases.ALL_CASES, ids=lambda c: c.__name__)
def test_reference_known_answers_on_oracle(orc, case):
    case(OracleApi(orc))


def test_rng_matches_reference(orc, ref):
    for seed in (0, 1, 42, 2**63 + 5):
        a, b = orc.rng(seed), ref.rng(seed)
        for _ in range(50):
            assert a.next_u64() == b.next_u64()
        for _ in range(21):
            assert a.next_gaussian(0.3, 2.0) == b.next_gaussian(0.3, 2.0)
            assert a.next_unit() == b.next_unit()
            assert a.next_below(97) == b.next_below(97)
    assert orc.rng(9).gaussian_f32(1001).tobytes() == ref.rng(9).gaussian_f32(1001).tobytes()


def test_oracle_bitwise_vs_reference(orc, ref):
    rs = np.random.default_rng(123)
    for _ in range(120):
        n = int(rs.integers(1, 160))
        dim = int(rs.choice([1, 2, 5, 8, 16, 64]))
        heads = int(rs.choice([h for h in (1, 2, 4) if dim % h == 0]))
        k = int(rs.integers(1, n + 3))
        lam = float(rs.choice([0.0, 1.0, rs.random()]))
        cloud = (rs.standard_normal((n, dim)) * rs.choice([0.01, 1.0, 30.0])).astype(np.float32)
        q = rs.standard_normal(dim).astype(np.float32)
        a1 = orc.attention_scores_points(cloud, q, heads)
        a2 = ref.attention_scores_points(cloud, q, heads)
        assert a1.tobytes() == a2.tobytes()
        i1, s1 = orc.select_landmarks_points(cloud, a1, k, lam)
        i2, s2 = ref.select_landmarks_points(cloud, a2, k, lam)
        assert i1.tobytes() == i2.tobytes() and s1.tobytes() == s2.tobytes()
        sel = i1[: max(1, len(i1) // 2)]
        assert orc.coverage_scores_points(cloud, sel).tobytes() == ref.coverage_scores_points(cloud, sel).tobytes()
        assert orc.coverage_scores_points(cloud, []).tobytes() == ref.coverage_scores_points(cloud, []).tobytes()
        assert orc.hausdorff_to_subset(cloud, i1) == ref.hausdorff_to_subset(cloud, i1)
        if len(i1) >= 2 and n >= 2:
            assert orc.mean_pairwise_reduction_subset(cloud, i1) == ref.mean_pairwise_reduction_subset(cloud, i1)
            assert orc.mean_pairwise_reduction(cloud, cloud[i1]) == ref.mean_pairwise_reduction(cloud, cloud[i1])
        assert orc.hausdorff_distance(cloud, cloud[i1]) == ref.hausdorff_distance(cloud, cloud[i1])
        H = heads
        dk = dim // H
        m = int(rs.integers(1, 40))
        kk = rs.standard_normal(m * dim).astype(np.float32)
        vv = rs.standard_normal(m * dim).astype(np.float32)
        assert orc.attend(q, kk, vv, m, H, dk).tobytes() == ref.attend(q, kk, vv, m, H, dk).tobytes()


def test_oracle_generators_vs_reference(orc, ref):
    for seed in (42, 43, 77):
        ro, rr = orc.rng(seed), ref.rng(seed)
        c1 = orc.make_clustered_cloud(ro, 256, 8, 5, 6.0, 0.5)
        c2 = ref.make_clustered_cloud(rr, 256, 8, 5, 6.0, 0.5)
        for x, y in zip(c1, c2):
            assert x.tobytes() == y.tobytes()
        assert np.array_equal(orc.random_subset(ro, 256, 16), ref.random_subset(rr, 256, 16))


def _golden(name):
    return np.load(os.path.join(GOLDEN, name))


def test_golden_small_cases(orc):
    g = _golden("select_small.npz")
    for c in range(len(g["seed"])):
        n, dim, k, lam, heads = (int(g["n"][c]), int(g["dim"][c]), int(g["k"][c]), float(g["lam"][c]),
                                 int(g["heads"][c]))
        r = orc.rng(int(g["seed"][c]))
        cloud = r.gaussian_f32(n * dim, 0.0, 2.0).reshape(n, dim)
        q = r.gaussian_f32(dim)
        sl = lambda key: g[key][g[key + "_off"][c]:g[key + "_off"][c + 1]]  # noqa: E731
        a = orc.attention_scores_points(cloud, q, heads)
        assert a.tobytes() == sl("attn").tobytes()
        idx, sc = orc.select_landmarks_points(cloud, a, k, lam)
        assert idx.tobytes() == sl("idx").tobytes() and sc.tobytes() == sl("scores").tobytes()
        cov = orc.coverage_scores_points(cloud, idx[: max(1, len(idx) // 2)])
        assert cov.tobytes() == sl("cov").tobytes()


@pytest.mark.parametrize("name", ["cfg1_points.npz", "cfg2_group.npz"])
def test_golden_group_cases(orc, name):
    g = _golden(name)
    keys, _, queries = oracle.synthetic_group(orc, int(g["seed"]), int(g["L"]), int(g["dim"]), int(g["n_q"]))
    a = oracle.group_attention(orc, keys, queries)
    assert a.tobytes() == g["attn"].tobytes()
    idx, sc = orc.select_landmarks_points(keys, a, int(g["k"]), float(g["lam"]))
    assert idx.tobytes() == g["idx"].tobytes() and sc.tobytes() == g["scores"].tobytes()


def test_golden_attend(orc):
    g = _golden("attend.npz")
    for c, (seed, n, H, dk) in enumerate(g["cases"]):
        r = orc.rng(int(seed))
        dm = int(H * dk)
        q = r.gaussian_f32(dm)
        kk = r.gaussian_f32(int(n) * dm)
        vv = r.gaussian_f32(int(n) * dm)
        out = orc.attend(q, kk, vv, int(n), int(H), int(dk))
        assert out.tobytes() == g["out"][g["off"][c]:g["off"][c + 1]].tobytes()


def test_golden_clustered_and_bench_landmarks(orc):
    g = _golden("clustered.npz")
    for s in range(3):
        r = orc.rng(42 + s)
        clusters = 2 + r.next_below(7)
        cloud, q, _ = orc.make_clustered_cloud(r, 256, 8, clusters, 6.0, 0.5)
        assert cloud.tobytes() == g[f"cloud{s}"].tobytes() and q.tobytes() == g[f"query{s}"].tobytes()
        a = orc.attention_scores_points(cloud, q, 2)
        idx, sc = orc.select_landmarks_points(cloud, a, 16, 0.5)
        assert idx.tobytes() == g[f"idx{s}"].tobytes() and sc.tobytes() == g[f"scores{s}"].tobytes()
        assert np.array_equal(orc.random_subset(r, 256, 16), g[f"random{s}"])
        assert orc.hausdorff_to_subset(cloud, idx) == float(g[f"haus{s}"])
        assert orc.mean_pairwise_reduction_subset(cloud, idx) == float(g[f"mpr{s}"])
    # bench_landmarks (harness/bench.cpp:330-425) re-run on the oracle: AC4 win rate
    with open(os.path.join(GOLDEN, "bench_landmarks.json")) as f:
        exp = json.load(f)["parameters"]
    wins, mh, mr = 0, 0.0, 0.0
    for s in range(100):
        r = orc.rng(42 + s)
        clusters = 2 + r.next_below(7)
        cloud, q, _ = orc.make_clustered_cloud(r, 256, 8, clusters, 6.0, 0.5)
        a = orc.attention_scores_points(cloud, q, 2)
        hyb, _ = orc.select_landmarks_points(cloud, a, 16, 0.5)
        orc.select_landmarks_points(cloud, a, 16, 0.0)
        rnd = orc.random_subset(r, 256, 16)
        wins += orc.hausdorff_to_subset(cloud, hyb) <= orc.hausdorff_to_subset(cloud, rnd)
        mh += orc.mean_pairwise_reduction_subset(cloud, hyb)
        mr += orc.mean_pairwise_reduction_subset(cloud, rnd)
    assert wins / 100 == exp["hybrid_win_rate"]
    assert mh / 100 == exp["mean_pairwise_reduction_hybrid"]
    assert mr / 100 == exp["mean_pairwise_reduction_random"]


def test_gate_oracle_bitwise_vs_reference(orc, ref):
    """gate.cpp:27-43: the C restatement == the unmodified reference, bit for bit, plus
    the reference's own known answers (test_gate.cpp:33-70)."""
    r = orc.rng(21)
    for dim in (1, 3, 64, 128, 1000):
        for _ in range(20):
            a, b = r.gaussian_f32(dim), r.gaussian_f32(dim)
            assert orc.gate_score(a, b) == ref.gate_score(a, b)
            assert orc.gate_score(a, -a) == ref.gate_score(a, -a)  # clamp side
    f = np.float32
    assert abs(orc.gate_score(np.array([0.4, -1.0, 2.0], f), np.array([0.4, -1.0, 2.0], f)) - 1.0) <= 1e-12
    assert orc.gate_score(np.array([1, 0, 0], f), np.array([0, 2, 0], f)) == 0.0
    assert abs(orc.gate_score(np.array([1, 2, 2], f), np.array([2, 1, 2], f)) - 8.0 / 9.0) <= 1e-12
    h, t = np.zeros(8, f), np.zeros(8, f)
    h[0] = 1.0
    t[:4] = 1.0
    assert orc.gate_score(h, t) == 0.5
    for be in (orc, ref):
        with pytest.raises(oracle.OracleError) as e:
            be.gate_score(np.zeros(4, f), np.array([1, 0, 0, 0], f))
        assert e.value.code == 7  # degenerate_input_error


def test_batched_decode_oracle_is_attend_per_q_head(orc, ref):
    """orc_decode_attend_agents (the checker of the batched decode) == the
    reference's own kernels::attend (n_heads = 1) called per (agent, layer,
    q-head) over [synapse rows || private rows], bit for bit, on ragged tails
    (empty tail included)."""
    rs = np.random.default_rng(3)
    N, Lr, H, Q, dk, k, tc = 5, 2, 2, 6, 16, 9, 7
    sk = rs.standard_normal((Lr, H, k, dk), dtype=np.float32)
    sv = rs.standard_normal((Lr, H, k, dk), dtype=np.float32)
    tk = rs.standard_normal((N, Lr, H, tc, dk), dtype=np.float32)
    tv = rs.standard_normal((N, Lr, H, tc, dk), dtype=np.float32)
    tl = np.array([0, 7, 3, 1, 5], np.int32)
    q = rs.standard_normal((N, Lr, Q, dk), dtype=np.float32)
    got = orc.decode_attend(sk, sv, tk, tv, tl, q, n_threads=3)
    back = ref if ref is not None else orc
    for a in range(N):
        for l in range(Lr):
            for h in range(Q):
                g = h // (Q // H)
                kk = np.concatenate([sk[l, g], tk[a, l, g, :tl[a]]])
                vv = np.concatenate([sv[l, g], tv[a, l, g, :tl[a]]])
                exp = back.attend(q[a, l, h], kk, vv, k + int(tl[a]), 1, dk)
                assert got[a, l, h].tobytes() == exp.tobytes(), (a, l, h)
