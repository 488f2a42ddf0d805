"""One selection launch for ncu (tools only)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd  # noqa: E402

G, L, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1, 8192, 164)))
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
keys = torch.randn(G, L, 64, device="cuda", generator=g)
q = torch.randn(G, 7, 64, device="cuda", generator=g)
a = cxd.attention_grouped(keys, q)
cxd.select_grouped(keys, a, k, 0.5, 0)
torch.cuda.synchronize()
print("ok")
