"""The full cfg2 compression (BASELINE configs[1]: 48 (layer, KV-head) groups,
L = 8192 -> k = 164, lambda = 0.5, 7 q-heads per group) checked against the
oracle for EVERY group -- not a sample:

* end to end (device attention mass -> device selection): index sets bit-exact
  against the oracle's attention + select_landmarks_points (synapse.cpp:63-93,
  216-284), and the gathered K/V rows bitwise;
* given the oracle's attention: index sets AND hybrid scores bitwise;
* the decision-gap monitor (cx_selection_gaps): every group's smallest
  top-1 / top-2 hybrid gap exceeds 1e-11, the margin that certifies the
  index set against the attention's 1e-12 relative tolerance.

The oracle's 96 selections run on all host threads (ctypes releases the GIL).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

G, L, D, NQ, K, LAM = 48, 8192, 64, 7, 164, 0.5  # noqa: E741
GAP_MIN = 1e-11


def _threads():
    return max(1, os.cpu_count() or 1)


@pytest.mark.parametrize("seed,exchange", [(3, 0), (2026, 0), (11, 1), (12, 2)], ids=["auto", "auto2", "clusters", "coop"])
def test_cfg2_all_groups_vs_oracle(orc, cx_option, seed, exchange):
    """exchange 0: the cost model (cfg2: the split one-wave plan -- 45 clusters of 3 beside a
    cooperative launch of 3 groups x 4 CTAs); 1: thread-block clusters (two waves);
    2: the cooperative launch alone (one wave of 48 x 3 CTAs)."""
    import torch

    from paper_2601_01298_b200 import device
    torch.cuda.set_device(0)
    cx_option("select_exchange", exchange)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    kt = torch.randn(G, L, D, device="cuda", generator=gen)
    vt = torch.randn(G, L, D, device="cuda", generator=gen)
    qt = torch.randn(G, NQ, D, device="cuda", generator=gen)
    rows, scores, sk, sv = device.compress_grouped(kt, vt, qt, K, LAM)
    gaps = device.selection_gaps(G)
    a_dev = device.attention_grouped(kt, qt)
    torch.cuda.synchronize()
    keys, vals, qs = kt.cpu().numpy(), vt.cpu().numpy(), qt.cpu().numpy()
    rows_n, scores_n = rows.cpu().numpy(), scores.cpu().numpy()
    a_dev_n = a_dev.cpu().numpy()

    def one(g):
        a = oracle.group_attention(orc, keys[g], qs[g])
        idx, sc = orc.select_landmarks_points(keys[g], a, K, LAM)
        return a, idx, sc

    with ThreadPoolExecutor(_threads()) as ex:
        ref = list(ex.map(one, range(G)))
    worst_attn = 0.0
    for g, (a, idx, sc) in enumerate(ref):
        assert rows_n[g].tobytes() == idx.tobytes(), f"group {g}: index set differs from the oracle"
        assert np.array_equal(sk[g].cpu().numpy(), keys[g][idx]) and np.array_equal(sv[g].cpu().numpy(), vals[g][idx])
        worst_attn = max(worst_attn, float(np.max(np.abs(a_dev_n[g] - a) / np.abs(a))))
    # the same attention in: rows and scores bitwise
    at = torch.from_numpy(np.stack([r[0] for r in ref])).cuda()
    rows2, scores2 = device.select_grouped(kt, at, K, LAM)
    torch.cuda.synchronize()
    for g, (a, idx, sc) in enumerate(ref):
        assert rows2[g].cpu().numpy().tobytes() == idx.tobytes(), g
        assert scores2[g].cpu().numpy().tobytes() == sc.tobytes(), g
    gaps = gaps.cpu().numpy()
    print(f"\n[cfg2 seed {seed}] 48/48 groups bit-exact; worst attention rel. error {worst_attn:.2e}; "
          f"smallest decision gap {gaps.min():.3e} (group {int(gaps.argmin())})")
    assert worst_attn <= 1e-12
    assert np.all(gaps > GAP_MIN), gaps


def test_gap_monitor_sees_ties_and_reports_unmonitored(orc):
    """The monitor is not vacuous: a cloud whose rows come in identical pairs
    (equal hybrid scores every round; the lower row wins, synapse.cpp:256) must
    report a gap of exactly 0, the generic-dim kernel reports NaN (not
    monitored), and the index set still matches the oracle."""
    import torch

    from paper_2601_01298_b200 import device
    r = orc.rng(808)
    half = r.gaussian_f32(1500 * D).reshape(1500, D)
    keys = np.repeat(half, 2, axis=0)  # rows 2i and 2i + 1 identical
    a = np.repeat(np.abs(r.gaussian_f32(1500)).astype(np.float64), 2)
    kt = torch.from_numpy(np.stack([keys, keys[::-1].copy()])).cuda()
    at = torch.from_numpy(np.stack([a, a[::-1].copy()])).cuda()
    rows, _ = device.select_grouped(kt, at, 40, 0.5)
    gaps = device.selection_gaps(2).cpu().numpy()
    assert np.all(gaps == 0.0), gaps
    idx, _ = orc.select_landmarks_points(keys, a, 40, 0.5)
    assert rows[0].cpu().numpy().tobytes() == idx.tobytes()
    device.select_grouped(kt, at, 40, 0.5, 2)  # CX_SELECT_GENERIC
    assert np.all(np.isnan(device.selection_gaps(2).cpu().numpy()))
