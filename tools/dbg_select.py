"""Debug harness (tools only): compare the device selection against the oracle
on the golden small cases and random dim-64 clouds, per flag setting."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2601_01298_b200 import device as cxd  # noqa: E402

orc = oracle.load()
torch.cuda.set_device(0)
g = np.load(os.path.join(ROOT, "tests", "golden", "select_small.npz"))
bad = {0: 0, 1: 0, 2: 0}
for c in range(len(g["seed"])):
    n, dim, k, lam, heads = (int(g["n"][c]), int(g["dim"][c]), int(g["k"][c]), float(g["lam"][c]), int(g["heads"][c]))
    if dim != 64:
        continue
    r = orc.rng(int(g["seed"][c]))
    cloud = r.gaussian_f32(n * dim, 0.0, 2.0).reshape(n, dim)
    att = g["attn"][g["attn_off"][c]:g["attn_off"][c + 1]]
    exp = g["idx"][g["idx_off"][c]:g["idx_off"][c + 1]]
    kt = torch.from_numpy(cloud).cuda()[None]
    at = torch.from_numpy(att).cuda()[None]
    for fl in (0, 1, 2):
        rows, _ = cxd.select_grouped(kt, at, k, lam, fl)
        got = rows.cpu().numpy()[0]
        if not np.array_equal(got, exp):
            bad[fl] += 1
            if bad[fl] <= 3:
                print(f"case {c} n={n} k={k} lam={lam:.3f} flags={fl}: got {got[:12]} exp {exp[:12]}")
print("mismatches per flag", bad)
rs = np.random.default_rng(5)
bad = {0: 0, 1: 0}
for t in range(40):
    n = int(rs.integers(1, 3000))
    k = int(rs.integers(1, min(n, 200) + 1))
    lam = float(rs.random())
    cloud = rs.standard_normal((n, 64)).astype(np.float32)
    att = rs.random(n)
    idx, _ = orc.select_landmarks_points(cloud, att, k, lam)
    kt = torch.from_numpy(cloud).cuda()[None]
    at = torch.from_numpy(att).cuda()[None]
    for fl in (0, 1):
        rows, _ = cxd.select_grouped(kt, at, k, lam, fl)
        got = rows.cpu().numpy()[0]
        if not np.array_equal(got, idx):
            bad[fl] += 1
            if bad[fl] <= 3:
                d = np.nonzero(got != idx)[0]
                print(f"rand {t} n={n} k={k} lam={lam:.3f} flags={fl}: first diff at {d[:5]} got {got[d[:5]]} exp {idx[d[:5]]}")
print("random mismatches per flag", bad)
