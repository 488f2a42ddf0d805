"""Selection timing, cluster kernels (d = 64 / 128) vs the generic-dim kernel (reference mode clouds: d_model = n_heads * d_k)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
for G, L, d, k in [(1, 8192, 128, 164), (1, 2048, 64, 40), (1, 8192, 64, 164), (1, 7168, 128, 143)]:
    keys = torch.randn(G, L, d, device="cuda", generator=g)
    a = torch.rand(G, L, device="cuda", generator=g, dtype=torch.float64)
    for flags, name in [(0, "cluster"), (2, "generic")]:
        for _ in range(2):
            cxd.select_grouped(keys, a, k, 0.5, flags)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            cxd.select_grouped(keys, a, k, 0.5, flags)
        e1.record(); torch.cuda.synchronize()
        print(f"G={G} L={L} d={d} k={k} {name}: {e0.elapsed_time(e1)/3:.3f} ms")
