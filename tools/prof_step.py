"""One cfg2 compression (48 groups, L=8192, k=164) + one N-agent decode step,
for ncu captures (tools only; timing comes from bench.py)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--groups", type=int, default=48)
ap.add_argument("--agents", type=int, default=1000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--what", default="both")  # both = compress + decode + inject
a = ap.parse_args()
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
if a.what in ("both", "compress"):
    keys = torch.randn(a.groups, 8192, 64, device="cuda", generator=g)
    vals = torch.randn(a.groups, 8192, 64, device="cuda", generator=g)
    q = torch.randn(a.groups, 7, 64, device="cuda", generator=g)
    for _ in range(a.reps):
        cxd.compress_grouped(keys, vals, q, 164, 0.5)
    torch.cuda.synchronize()
if a.what in ("both", "decode"):
    N = a.agents
    sk = torch.randn(24, 2, 164, 64, device="cuda", generator=g)
    sv = torch.randn(24, 2, 164, 64, device="cuda", generator=g)
    tk = torch.randn(N, 24, 2, 33, 64, device="cuda", generator=g)
    tv = torch.randn(N, 24, 2, 33, 64, device="cuda", generator=g)
    tl = torch.full((N,), 32, dtype=torch.int32, device="cuda")
    nk = torch.randn(N, 24, 2, 64, device="cuda", generator=g)
    nv = torch.randn(N, 24, 2, 64, device="cuda", generator=g)
    qq = torch.randn(N, 24, 14, 64, device="cuda", generator=g)
    o = torch.empty_like(qq)
    for _ in range(a.reps):
        cxd.decode_step(sk, sv, tk, tv, tl, qq, o, nk, nv)
    torch.cuda.synchronize()
if a.what in ("both", "inject"):  # Referential Injection append (cfg5: 16-token block into the river cache)
    from paper_2601_01298_b200.injector import inject_dev
    from paper_2601_01298_b200.model import KvCache, ModelConfig
    cfg = ModelConfig(n_layers=24, n_heads=2, d_model=128, d_k=64, max_positions=16384)
    river = KvCache(cfg, capacity=8192 + 64)
    pk = torch.randn(24, 8192, 128, device="cuda", generator=g)
    river.append_context_dev(pk.data_ptr(), pk.data_ptr(), 0, 8192, torch.cuda.current_stream().cuda_stream)
    tk = torch.randn(24, 16, 128, device="cuda", generator=g)
    for r in range(a.reps):
        inject_dev(river, tk.data_ptr(), tk.data_ptr(), 9000 + 16 * r, 16, 24, 128, r, 0,
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
print("ok")
