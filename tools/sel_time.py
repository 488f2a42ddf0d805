"""cfg2 selection latency (48 groups, L=8192, k=164) per plan (tools only):
python tools/sel_time.py [exchange] [C]"""
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
if len(sys.argv) > 1:
    cxd.set_option("select_exchange", int(sys.argv[1]))
if len(sys.argv) > 2:
    cxd.set_option("select_cluster", int(sys.argv[2]))
if os.environ.get("STREAM"):  # run on a non-default (optionally high-priority) stream
    torch.cuda.set_stream(torch.cuda.Stream(priority=int(os.environ["STREAM"])))
KS = int(os.environ.get("K", "164"))
ref = cxd.select_grouped(keys, a, KS, 0.5)
flush = torch.empty(64 << 20, device="cuda")
ts = []
for _ in range(10):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    r = cxd.select_grouped(keys, a, KS, 0.5)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    assert torch.equal(r[0], ref[0])
ts.sort()
print(f"exchange={sys.argv[1] if len(sys.argv) > 1 else 'auto'} C={sys.argv[2] if len(sys.argv) > 2 else 'auto'}: "
      f"median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f}")
