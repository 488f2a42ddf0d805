"""One cfg2 selection (48 groups, L=8192, k=164) for ncu captures (tools only)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd  # noqa: E402

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
G = int(os.environ.get("G", "48"))
keys = torch.randn(G, 8192, 64, device="cuda", generator=g)
q = torch.randn(G, 7, 64, device="cuda", generator=g)
a = cxd.attention_grouped(keys, q)
if os.environ.get("IMPL"):
    cxd.set_option("select_impl", os.environ["IMPL"])
if os.environ.get("C"):
    cxd.set_option("select_cluster", int(os.environ["C"]))
for _ in range(int(os.environ.get("REPS", "1"))):
    cxd.select_grouped(keys, a, 164, 0.5)
torch.cuda.synchronize()
print("ok")
