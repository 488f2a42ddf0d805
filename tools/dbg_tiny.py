import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle
from paper_2601_01298_b200 import device as cxd
orc = oracle.load()
torch.cuda.set_device(0)
g = np.load(os.path.join(ROOT, "tests", "golden", "select_small.npz"))
c = int(sys.argv[1]) if len(sys.argv) > 1 else 7
n, dim, k, lam = int(g["n"][c]), int(g["dim"][c]), int(g["k"][c]), float(g["lam"][c])
r = orc.rng(int(g["seed"][c]))
cloud = r.gaussian_f32(n * dim, 0.0, 2.0).reshape(n, dim)
att = g["attn"][g["attn_off"][c]:g["attn_off"][c + 1]]
for kk in (1, 2, 3, k):
    idx, sc = orc.select_landmarks_points(cloud, att, kk, lam)
    print("k", kk, "oracle sorted", idx[:8], sc[:8])
    rows, scores = cxd.select_grouped(torch.from_numpy(cloud).cuda()[None], torch.from_numpy(att).cuda()[None], kk, lam, 1)
    print("k", kk, "gpu", rows.cpu().numpy()[0][:8], scores.cpu().numpy()[0][:8])
