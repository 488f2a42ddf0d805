"""Micro-timing of the selection kernel across shapes (tools only)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd  # noqa: E402

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


shapes = [(1, 8192, 1), (1, 8192, 164), (7, 8192, 164), (48, 8192, 1), (48, 8192, 164), (48, 8192, 41),
          (1, 2048, 40), (1, 32768, 656)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
for G, L, k in shapes:
    keys = torch.randn(G, L, 64, device="cuda", generator=g)
    q = torch.randn(G, 7, 64, device="cuda", generator=g)
    a = cxd.attention_grouped(keys, q)
    ta = t(lambda: cxd.attention_grouped(keys, q))
    tf = t(lambda: cxd.select_grouped(keys, a, k, 0.5, 0))
    te = t(lambda: cxd.select_grouped(keys, a, k, 0.5, 1))
    print(f"G={G:3d} L={L:6d} k={k:4d}  attention {ta:8.3f} ms  select(filter) {tf:8.3f} ms  "
          f"select(exact) {te:8.3f} ms  per-round {1000*tf/max(k,1):7.2f} us", flush=True)
