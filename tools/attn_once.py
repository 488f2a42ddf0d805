"""Attention mass of the cfg2 shape once per implementation (tools only; for ncu launch lists)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd
g = torch.Generator(device="cuda").manual_seed(5)
k = torch.randn(48, 8192, 64, device="cuda", generator=g); q = torch.randn(48, 7, 64, device="cuda", generator=g)
for impl in (0, 1, 0, 1):
    cxd.set_option("attn_impl", impl)
    cxd.attention_grouped(k, q)
torch.cuda.synchronize()
print("ok")
