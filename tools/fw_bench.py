"""forward_step cost on the cfg5 river (24 layers x d_model 128, L context rows):
device time per token (CUDA events) and host issue time.  Usage:
python tools/fw_bench.py [L] [n_tokens]   (STREAM=1: on a created stream, where the step
replays as a captured CUDA graph; the default stream issues the launches directly)"""
import os
import sys
import time

import torch

sys.path.insert(0, __import__("os").environ.get("CX_PKG_ROOT") or __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2601_01298_b200 import runtime as rt  # noqa: E402
from paper_2601_01298_b200.model import KvCache, ModelConfig  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = ModelConfig(n_layers=24, n_heads=2, d_model=128, d_k=64, vocab_size=256, max_positions=L + 4096)
w = rt.Weights(cfg, rt.random_flat_weights(cfg, 7))
river = KvCache(cfg, capacity=L + n + 64)
pk = torch.randn(24, L, 128, device="cuda")
pv = torch.randn(24, L, 128, device="cuda")
torch.cuda.synchronize()
river.append_context_dev(pk.data_ptr(), pv.data_ptr(), 0, L)
torch.cuda.synchronize()
logits = torch.empty(256, device="cuda")
stream = torch.cuda.Stream() if os.environ.get("STREAM") == "1" else torch.cuda.current_stream()
torch.cuda.set_stream(stream)
for i in range(5):
    rt.forward_step_dev(w, [river], [i], [L + i], logits=logits)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for i in range(n):
    rt.forward_step_dev(w, [river], [i % 256], [L + 5 + i], logits=logits)
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"L={L}: device {e0.elapsed_time(e1) / n * 1e3:.1f} us/token, host issue {(t1 - t0) / n * 1e6:.1f} us/token")
