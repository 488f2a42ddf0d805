"""Selection timing per group count with the launch configuration (tools only)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
for G in [int(x) for x in (sys.argv[1:] or ["22", "26", "48"])]:
    keys = torch.randn(G, 8192, 64, device="cuda", generator=g)
    q = torch.randn(G, 7, 64, device="cuda", generator=g)
    a = cxd.attention_grouped(keys, q)
    for _ in range(2):
        cxd.select_grouped(keys, a, 164, 0.5)
    torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); cxd.select_grouped(keys, a, 164, 0.5); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"G={G}: select {min(ts):.3f} ms (min of 4), {sorted(ts)}", flush=True)
