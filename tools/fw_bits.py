"""Logits of a fixed forward_step sequence (tools only): python tools/fw_bits.py OUT.pt;
compare two builds' files with --cmp A.pt B.pt (bitwise)."""
import os
import sys

import torch

if sys.argv[1] == "--cmp":
    a, b = torch.load(sys.argv[2]), torch.load(sys.argv[3])
    print("bitwise equal:", all(torch.equal(x, y) for x, y in zip(a, b)), [float((x - y).abs().max()) for x, y in zip(a, b)])
    sys.exit(0)
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import runtime as rt  # noqa: E402
from paper_2601_01298_b200.model import KvCache, ModelConfig  # noqa: E402

cfg = ModelConfig(n_layers=4, n_heads=2, d_model=128, d_k=64, vocab_size=256, max_positions=8192)
w = rt.Weights(cfg, rt.random_flat_weights(cfg, 5))
g = torch.Generator(device="cuda").manual_seed(9)
L0 = 300
pk = torch.randn(4, L0, 128, device="cuda", generator=g)
pv = torch.randn(4, L0, 128, device="cuda", generator=g)
outs = []
for nb in (1, 2, 3):
    caches = [KvCache(cfg, capacity=L0 + 64) for _ in range(nb)]
    torch.cuda.synchronize()
    for c in caches:
        c.append_context_dev(pk.data_ptr(), pv.data_ptr(), 0, L0)
    torch.cuda.synchronize()
    lg = torch.empty(40, nb, 256, device="cuda")
    hd = torch.empty(40, nb, 128, device="cuda")
    for t in range(40):
        rt.forward_step_dev(w, caches, [(5 * t + b) % 256 for b in range(nb)], [L0 + t] * nb, logits=lg[t], hidden=hd[t])
    torch.cuda.synchronize()
    outs += [lg.cpu(), hd.cpu()]
torch.save(outs, sys.argv[1])
print("saved", sys.argv[1])
