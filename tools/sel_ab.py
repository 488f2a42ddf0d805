"""cfg2 compression / selection timing for A/B of library variants (tools only):
CX_PKG_ROOT=.variants/NAME python tools/sel_ab.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd  # noqa: E402

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
G = 48
keys = torch.randn(G, 8192, 64, device="cuda", generator=g)
vals = torch.randn(G, 8192, 64, device="cuda", generator=g)
q = torch.randn(G, 7, 64, device="cuda", generator=g)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
a = cxd.attention_grouped(keys, q)
ref = cxd.compress_grouped(keys, vals, q, 164, 0.5)[0].clone()


def timed(fn, n=10):
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for _ in range(2):
    cxd.compress_grouped(keys, vals, q, 164, 0.5)
comp = timed(lambda: cxd.compress_grouped(keys, vals, q, 164, 0.5))
sel = timed(lambda: cxd.select_grouped(keys, a, 164, 0.5))
rows = cxd.compress_grouped(keys, vals, q, 164, 0.5)[0]
print(f"{os.environ.get('CX_PKG_ROOT', 'main')}: compress {comp:.3f} ms  select {sel:.3f} ms  same_rows={bool(torch.equal(rows, ref))}")
