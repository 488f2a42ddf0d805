"""e2e compression timing (host buffers) per chunking (tools only; CX_E2E_CHUNKS)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd
torch.cuda.set_device(0)
G, L, D, K = 48, 8192, 64, 164
hk = torch.randn(G, L, D).pin_memory(); hv = torch.randn(G, L, D).pin_memory(); hq = torch.randn(G, 7, D).pin_memory()
out = (torch.empty(G, K, dtype=torch.int64).pin_memory(), torch.empty(G, K, dtype=torch.float64).pin_memory(),
       torch.empty(G, K, D).pin_memory(), torch.empty(G, K, D).pin_memory())
for ch in sys.argv[1:] or ["default"]:
    if ch == "default":
        os.environ.pop("CX_E2E_CHUNKS", None)
    else:
        os.environ["CX_E2E_CHUNKS"] = ch
    for _ in range(2):
        cxd.compress_grouped_host(hk, hv, hq, K, 0.5, out=out)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        cxd.compress_grouped_host(hk, hv, hq, K, 0.5, out=out)
    e1.record(); torch.cuda.synchronize()
    print(f"{ch:>16}: {e0.elapsed_time(e1) / 5:.3f} ms")
