"""One decode configuration, a few launches (tools only; for ncu)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd
N = int(os.environ.get("N", "1000"))
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
sk = torch.randn(24, 2, 164, 64, device="cuda", generator=g); sv = torch.randn_like(sk)
tk = torch.randn(N, 24, 2, 33, 64, device="cuda", generator=g); tv = torch.randn_like(tk)
tl = torch.full((N,), 32, dtype=torch.int32, device="cuda")
nk = torch.randn(N, 24, 2, 64, device="cuda", generator=g); nv = torch.randn_like(nk)
q = torch.randn(N, 24, 14, 64, device="cuda", generator=g); o = torch.empty_like(q)
for _ in range(int(os.environ.get("REPS", "3"))):
    cxd.decode_step(sk, sv, tk, tv, tl, q, o, nk, nv)
torch.cuda.synchronize()
print("ok")
