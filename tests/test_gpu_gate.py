"""The gate (gate.cpp:12-61) on the B200: the batched device form
(cx_gate_decide_dev) and the single-pair cortex:: API (cx_gate_score) against the
oracle, bit for bit, with the reference's edge cases (zero norms, exact threshold,
clamp, theta range)."""
import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cx():
    import torch
    torch.cuda.set_device(0)
    import paper_2601_01298_b200 as m
    return m


@pytest.fixture(scope="module")
def orc():
    return oracle.load()


def test_gate_decide_batched_matches_oracle(cx, orc):
    import torch
    from paper_2601_01298_b200 import device
    n, dim = 333, 128
    r = orc.rng(77)
    h = r.gaussian_f32(n * dim).reshape(n, dim)
    t = r.gaussian_f32(n * dim).reshape(n, dim)
    t[5] = h[5]            # self similarity
    t[6] = -h[6]           # -1 (clamp side)
    h[7] = 0.0             # degenerate
    t[8] = 0.0             # degenerate
    h[9] = 0.0; h[9, 0] = 1.0
    t[9] = 0.0; t[9, :4] = 1.0   # exactly 0.5
    theta = 0.5
    sc, acc, deg = device.gate_decide(torch.from_numpy(h).cuda(), torch.from_numpy(t).cuda(), theta)
    torch.cuda.synchronize()
    sc, acc, deg = sc.cpu().numpy(), acc.cpu().numpy(), deg.cpu().numpy()
    for i in range(n):
        try:
            exp = orc.gate_score(h[i], t[i])
        except oracle.OracleError as e:
            assert e.code == 7 and deg[i] and not acc[i] and math.isnan(sc[i]), i
            continue
        assert not deg[i]
        assert sc[i] == exp, (i, sc[i], exp)  # bitwise
        assert bool(acc[i]) == (exp >= theta)
    assert sc[9] == 0.5 and acc[9]
    assert deg[7] and deg[8]


def test_gate_strided_rows_and_theta(cx, orc):
    """Rows read through a stride (a slice of wider hidden states); theta outside [-1, 1]
    rejected before any work (gate.cpp:47-48)."""
    import torch
    from paper_2601_01298_b200 import device
    r = orc.rng(3)
    big_h = torch.from_numpy(r.gaussian_f32(40 * 200).reshape(40, 200)).cuda()
    big_t = torch.from_numpy(r.gaussian_f32(40 * 200).reshape(40, 200)).cuda()
    h, t = big_h[:, 10:74], big_t[:, 100:164]
    sc, acc, deg = device.gate_decide(h, t, -0.05)
    torch.cuda.synchronize()
    hn, tn = h.cpu().numpy(), t.cpu().numpy()
    for i in range(40):
        assert sc[i].item() == orc.gate_score(np.ascontiguousarray(hn[i]), np.ascontiguousarray(tn[i]))
        assert bool(acc[i]) == (sc[i].item() >= -0.05)
    with pytest.raises(cx.errors.precondition_error):
        device.gate_decide(h, t, 1.5)


def test_gate_single_pair_api(cx, orc):
    """cortex::gate_score / decide (gate.hpp:22-27) through the Python mirror."""
    f = np.float32
    r = orc.rng(11)
    for _ in range(25):
        a, b = r.gaussian_f32(64), r.gaussian_f32(64)
        assert cx.gate_score(a, b) == orc.gate_score(a, b)
    assert cx.gate_score(np.array([1, 0, 0], f), np.array([0, 2, 0], f)) == 0.0
    h, t = np.zeros(8, f), np.zeros(8, f)
    h[0] = 1.0
    t[:4] = 1.0
    assert cx.gate_score(h, t) == 0.5
    assert cx.decide(h, t, 0.5).accepted and not cx.decide(h, t, 0.5000001).accepted
    with pytest.raises(cx.errors.degenerate_input_error):
        cx.gate_score(np.zeros(4, f), np.array([1, 0, 0, 0], f))
    d = cx.decide(np.zeros(4, f), np.array([1, 0, 0, 0], f), 0.5, 7)
    assert d.degenerate and not d.accepted and math.isnan(d.score) and d.thought_id == 7
    assert d.csv_row() == "7,nan,0.5,0"
    with pytest.raises(cx.errors.precondition_error):
        cx.decide(h, h, 1.5)
    with pytest.raises(cx.errors.precondition_error):
        cx.gate_score(h, t[:4])
