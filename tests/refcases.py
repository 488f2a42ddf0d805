"""The reference's own known-answer tests for the synapse path, restated once
and run against any implementation with the point-level API:

  * the oracle (CPU, tests/test_oracle_pins.py) -- pins the restatement;
  * the B200 product (GPU, tests/test_gpu_parity.py) -- parity.

Sources (file:line under /root/reference/proj/tests):
  test_synapse.cpp:87-396, test_kernels.cpp:72-163, acceptance.cpp:147-187.

An ``api`` object provides: attention_scores_points, coverage_scores_points,
select_landmarks_points -> (idx, scores), hausdorff_distance,
hausdorff_to_subset, mean_pairwise_reduction, mean_pairwise_reduction_subset,
attend, softmax, argmax, rng(seed) (cortex::Rng), and error_kind(exc) -> reference type name.
"""
from __future__ import annotations

import math

import numpy as np


def _approx(a, b, eps=1e-12):
    # doctest::Approx(b).epsilon(eps): |a-b| < eps * (scale + max(|a|,|b|)), scale = 1
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def expect_error(api, kind, fn, *args):
    try:
        fn(*args)
    except Exception as e:  # noqa: BLE001
        got = api.error_kind(e)
        assert got == kind, f"expected {kind}, got {got}: {e}"
        return
    raise AssertionError(f"expected {kind}, nothing raised")


def topk_oracle(scores, k):
    """test_synapse.cpp:63-74 -- descending score, ties to the lower index."""
    idx = sorted(range(len(scores)), key=lambda i: (-scores[i], i))[: min(k, len(scores))]
    return np.asarray(sorted(idx), dtype=np.int64)


def random_cloud(rng, n, dim, spread=2.0):
    """test_synapse.cpp:76-83."""
    return rng.gaussian_f32(n * dim, 0.0, spread).reshape(n, dim)


def dist_oracle(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = 0.0
    for x, y in zip(a, b):
        d = x - y
        s += d * d
    return math.sqrt(s)


# ---- test_synapse.cpp --------------------------------------------------------

def case_uniform_attention(api):  # :87-94
    a = api.attention_scores_points(np.array([[0, 1], [0, 2], [0, -3]], np.float32), np.array([1, 0], np.float32), 1)
    assert len(a) == 3
    for v in a:
        assert _approx(v, 1.0 / 3.0)


def case_two_key_attention(api):  # :96-106
    a = api.attention_scores_points(np.array([[1, 0], [0, 1]], np.float32), np.array([1, 0], np.float32), 1)
    s = 1.0 / math.sqrt(2.0)
    z = math.exp(s) + 1.0
    assert _approx(a[0], math.exp(s) / z)
    assert _approx(a[1], 1.0 / z)


def case_per_head_sum(api):  # :108-128 (layer-1 keys of an 11-entry, 2-layer cache)
    rng = api.rng(31)
    rows = []
    for _ in range(11):
        k = rng.gaussian_f32(32)
        rng.gaussian_f32(32)  # values
        rows.append(k[16:32])
    q = rng.gaussian_f32(16)
    a = api.attention_scores_points(np.stack(rows), q, 4)
    assert abs(float(np.sum(a)) - 4) < 1e-6


def case_empty_attention(api):  # :130-135
    expect_error(api, "precondition_error", api.attention_scores_points, np.zeros((0, 2), np.float32),
                 np.array([1, 0], np.float32), 1)


def case_coverage(api):  # :137-163
    s = api.coverage_scores_points(np.array([[0, 0], [1, 0], [10, 0]], np.float32), [0])
    assert s[0] == 0.0 and _approx(s[1], 1.0) and _approx(s[2], 10.0)
    s = api.coverage_scores_points(np.array([[0, 1], [2, 3]], np.float32), [0, 1])
    assert s[0] == 0.0 and s[1] == 0.0
    s = api.coverage_scores_points(np.array([[0, 0], [4, 0]], np.float32), [])
    assert _approx(s[0], 2.0) and _approx(s[1], 2.0)


def case_saturation(api):  # :165-177 (point-level form)
    cloud = np.array([[0, 0], [1, 0], [2, 0], [3, 0]], np.float32)
    a = api.attention_scores_points(cloud, np.array([1, 0], np.float32), 1)
    idx, _ = api.select_landmarks_points(cloud, a, 9, 0.5)
    assert list(idx) == [0, 1, 2, 3]


def case_config_errors(api):  # :179-184
    cloud = np.array([[0, 0]], np.float32)
    expect_error(api, "config_error", api.select_landmarks_points, cloud, np.array([1.0]), 0, 0.5)
    expect_error(api, "config_error", api.select_landmarks_points, cloud, np.array([1.0]), 1, 1.5)
    expect_error(api, "precondition_error", api.select_landmarks_points, cloud, np.array([1.0, 2.0]), 1, 0.5)


def case_lambda0_topk(api):  # :186-197
    rng = api.rng(41)
    for _ in range(30):
        n = 1 + rng.next_below(64)
        k = 1 + rng.next_below(n)
        cloud = random_cloud(rng, n, 8)
        attn = np.array([rng.next_unit() for _ in range(n)])
        idx, _ = api.select_landmarks_points(cloud, attn, k, 0.0)
        assert np.array_equal(idx, topk_oracle(list(attn), k))


def case_ties(api):  # :199-204
    idx, _ = api.select_landmarks_points(np.array([[0, 0], [1, 1], [2, 2]], np.float32), np.array([0.5] * 3), 2, 0.0)
    assert list(idx) == [0, 1]


def case_two_clusters(api):  # :206-239
    pts = []
    for i in range(5):
        a = [10.0] * 16
        a[i] = 11.0
        pts.append(a)
        b = [-10.0] * 16
        b[i] = -9.0
        pts.append(b)
    cloud = np.array(pts, np.float32)
    idx, _ = api.select_landmarks_points(cloud, np.zeros(len(pts)), 2, 1.0)
    assert len(idx) == 2
    assert (cloud[idx[0]][2] > 0) != (cloud[idx[1]][2] > 0)
    best = math.inf
    for i in range(len(pts)):
        for j in range(i + 1, len(pts)):
            worst = 0.0
            for p in range(len(pts)):
                worst = max(worst, min(dist_oracle(cloud[p], cloud[i]), dist_oracle(cloud[p], cloud[j])))
            best = min(best, worst)
    assert _approx(api.hausdorff_to_subset(cloud, idx), best)


def case_incremental_equals_scratch(api):  # :241-288
    rng = api.rng(43)
    for _ in range(10):
        n = 10 + rng.next_below(50)
        k = 1 + rng.next_below(12)
        lam = rng.next_unit()
        cloud = random_cloud(rng, n, 6)
        attn = np.array([rng.next_unit() for _ in range(n)])
        selected, taken = [], [False] * n
        for _r in range(min(k, n)):
            cov = api.coverage_scores_points(cloud, selected)
            amin, amax, cmin, cmax = 1e300, -1e300, 1e300, -1e300
            for i in range(n):
                if taken[i]:
                    continue
                amin, amax = min(amin, attn[i]), max(amax, attn[i])
                cmin, cmax = min(cmin, cov[i]), max(cmax, cov[i])
            best, best_score = -1, -1.0
            for i in range(n):
                if taken[i]:
                    continue
                na = (attn[i] - amin) / (amax - amin) if amax > amin else 0.0
                nc = (cov[i] - cmin) / (cmax - cmin) if cmax > cmin else 0.0
                h = lam * nc + (1.0 - lam) * na
                if h > best_score:
                    best, best_score = i, h
            taken[best] = True
            selected.append(best)
        idx, _ = api.select_landmarks_points(cloud, attn, k, lam)
        assert list(idx) == sorted(selected)


def case_hausdorff(api):  # :323-352
    cloud = np.array([[0, 0], [10, 0]], np.float32)
    assert api.hausdorff_distance(cloud, cloud) == 0.0
    assert _approx(api.hausdorff_distance(cloud, np.array([[0, 0]], np.float32)), 10.0)
    expect_error(api, "precondition_error", api.hausdorff_distance, cloud, np.zeros((0, 2), np.float32))
    rng = api.rng(51)
    cloud = random_cloud(rng, 20, 6)
    rows = [2, 5, 9, 13, 17]
    worst = 0.0
    for i in range(20):
        worst = max(worst, min(dist_oracle(cloud[i], cloud[r]) for r in rows))
    assert _approx(api.hausdorff_distance(cloud, cloud[rows]), worst)
    assert _approx(api.hausdorff_to_subset(cloud, rows), worst)


def case_mean_pairwise(api):  # :354-396
    cloud = np.array([[0, 0], [1, 0], [2, 0], [3, 0]], np.float32)
    assert _approx(api.mean_pairwise_reduction_subset(cloud, [1, 2]), 1.0 - 1.0 / (10.0 / 6.0))
    assert abs(api.mean_pairwise_reduction_subset(cloud, [0, 1, 2, 3])) < 1e-5 * 1.0  # doctest::Approx(0.0)
    rng = api.rng(53)
    cloud = random_cloud(rng, 12, 5)
    rows = [1, 4, 7, 9]
    assert _approx(api.mean_pairwise_reduction(cloud, cloud[rows]), api.mean_pairwise_reduction_subset(cloud, rows))
    flat = np.full((5, 3), 2.0, np.float32)
    assert api.mean_pairwise_reduction_subset(flat, [0, 3]) == 0.0
    expect_error(api, "precondition_error", api.mean_pairwise_reduction_subset, flat, [0])


# ---- test_kernels.cpp:131-163 -------------------------------------------------

def case_attend(api):
    rng = api.rng(13)
    H, dk, L = 4, 8, 19
    dm = H * dk
    q = rng.gaussian_f32(dm)
    keys = rng.gaussian_f32(L * dm)
    values = rng.gaussian_f32(L * dm)
    out = api.attend(q, keys, values, L, H, dk)
    K = keys.reshape(L, dm).astype(np.float64)
    V = values.reshape(L, dm).astype(np.float64)
    for h in range(H):
        s = K[:, h * dk:(h + 1) * dk] @ q[h * dk:(h + 1) * dk].astype(np.float64) / math.sqrt(dk)
        p = np.exp(s - s.max())
        p /= p.sum()
        acc = p @ V[:, h * dk:(h + 1) * dk]
        for c in range(dk):
            assert abs(out[h * dk + c] - acc[c]) <= 1e-6 * max(1.0, abs(acc[c]))


# ---- test_kernels.cpp:72-114: softmax / argmax known answers --------------------

def case_softmax_uniform(api):  # :72-76
    p = api.softmax(np.full(7, 4.2))
    assert all(_approx(v, 1.0 / 7.0) for v in p)


def case_softmax_scalar(api):  # :78-90
    p = api.softmax(np.array([1.0, 2.0, 3.0]))
    e1, e2, e3 = math.exp(1.0 - 3.0), math.exp(2.0 - 3.0), 1.0
    z = e1 + e2 + e3
    assert abs(p[0] - e1 / z) < 1e-12 and abs(p[1] - e2 / z) < 1e-12 and abs(p[2] - e3 / z) < 1e-12
    assert abs(sum(p) - 1.0) < 1e-9


def case_softmax_gap(api):  # :92-101
    prev = 0.0
    for gap in range(1, 31):
        p = api.softmax(np.array([0.0, float(gap)]))
        assert p[1] > prev
        prev = p[1]
    assert prev > 1.0 - 1e-12


def case_softmax_errors(api):  # :103-110
    expect_error(api, "precondition_error", api.softmax, np.zeros(0))
    expect_error(api, "precondition_error", api.softmax, np.array([1.0, math.inf]))


def case_argmax_ties(api):  # :112-115
    assert api.argmax(np.array([0.5, 2.0, 2.0, -1.0], np.float32)) == 1


# ---- acceptance.cpp:147-187 (AC3) ---------------------------------------------

def paired_cluster_cloud(dim, per_cluster):
    cloud = np.zeros((2 * per_cluster, dim), np.float32)
    for i in range(per_cluster):
        cloud[2 * i, :] = 10.0
        cloud[2 * i, i] = 11.0
        cloud[2 * i + 1, :] = -10.0
        cloud[2 * i + 1, i] = -9.0
    return cloud


def case_ac3(api, trials=200):
    rng = api.rng(42)
    for _ in range(trials):
        n = 1 + rng.next_below(64)
        k = 1 + rng.next_below(n)
        cloud = rng.gaussian_f32(n * 16, 0.0, 2.0).reshape(n, 16)
        attn = np.array([rng.next_unit() for _ in range(n)])
        idx, _ = api.select_landmarks_points(cloud, attn, k, 0.0)
        assert np.array_equal(idx, topk_oracle(list(attn), k))

    def brute(cloud, rows):
        return max(min(dist_oracle(cloud[i], cloud[r]) for r in rows) for i in range(len(cloud)))

    for per in range(2, 7):
        cloud = paired_cluster_cloud(32, per)
        idx, _ = api.select_landmarks_points(cloud, np.zeros(len(cloud)), 2, 1.0)
        ours = brute(cloud, list(idx))
        best = min(brute(cloud, [i, j]) for i in range(len(cloud)) for j in range(i + 1, len(cloud)))
        assert ours == best


ALL_CASES = [
    case_uniform_attention, case_two_key_attention, case_per_head_sum, case_empty_attention, case_coverage,
    case_saturation, case_config_errors, case_lambda0_topk, case_ties, case_two_clusters,
    case_incremental_equals_scratch, case_hausdorff, case_mean_pairwise, case_attend, case_ac3,
    case_softmax_uniform, case_softmax_scalar, case_softmax_gap, case_softmax_errors, case_argmax_ties,
]
