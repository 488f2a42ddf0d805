"""cfg2 compression timings for A/B runs (tools only): device path (inputs in HBM, L2 flushed
between steps) and host-buffer path (cx_compress_grouped_host), as bench.py measures them.
CX_PKG_ROOT=.variants/NAME selects a variant build; TAG labels the line."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd  # noqa: E402

G, L, D, K, LAM, QPG = 48, 8192, 64, 164, 0.5, 7
torch.cuda.set_device(0)
for kv in filter(None, os.environ.get("OPTS", "").split(",")):  # e.g. OPTS=attn_impl=1
    cxd.set_option(kv.split("=")[0], int(kv.split("=")[1]))
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(1234)
keys = torch.randn(G, L, D, device=dev, generator=gen)
values = torch.randn(G, L, D, device=dev, generator=gen)
queries = torch.randn(G, QPG, D, device=dev, generator=gen)
out = (torch.empty(G, K, dtype=torch.int64, device=dev), torch.empty(G, K, dtype=torch.float64, device=dev),
       torch.empty(G, K, D, device=dev), torch.empty(G, K, D, device=dev))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(3):
    cxd.compress_grouped(keys, values, queries, K, LAM, out=out)
torch.cuda.synchronize()
times = []
for _ in range(int(os.environ.get("STEPS", "30"))):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cxd.compress_grouped(keys, values, queries, K, LAM, out=out)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
# the synapse must equal a plain gather of the selected rows
rows = out[0]
ref_k = torch.gather(keys, 1, rows.unsqueeze(-1).expand(G, K, D))
ref_v = torch.gather(values, 1, rows.unsqueeze(-1).expand(G, K, D))
ok = torch.equal(ref_k, out[2]) and torch.equal(ref_v, out[3])
hk, hv, hq = keys.cpu().pin_memory(), values.cpu().pin_memory(), queries.cpu().pin_memory()
h_out = (torch.empty(G, K, dtype=torch.int64).pin_memory(), torch.empty(G, K, dtype=torch.float64).pin_memory(),
         torch.empty(G, K, D).pin_memory(), torch.empty(G, K, D).pin_memory())
for _ in range(2):
    cxd.compress_grouped_host(hk, hv, hq, K, LAM, out=h_out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    cxd.compress_grouped_host(hk, hv, hq, K, LAM, out=h_out)
e1.record()
torch.cuda.synchronize()
e2e = e0.elapsed_time(e1) / 10
ok_h = all(torch.equal(a.cpu(), b) for a, b in zip(out, h_out))
a_t = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cxd.attention_grouped(keys, queries)
    e1.record()
    torch.cuda.synchronize()
    a_t.append(e0.elapsed_time(e1))
attn = cxd.attention_grouped(keys, queries)
s_t = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cxd.select_grouped(keys, attn, K, LAM)
    e1.record()
    torch.cuda.synchronize()
    s_t.append(e0.elapsed_time(e1))
print(f"{os.environ.get('TAG', '')}: centroid+selection {statistics.mean(s_t):.4f} ms, attention {statistics.mean(a_t) * 1e3:.1f} us, device {statistics.mean(times):.4f} ms (min {min(times):.4f}), "
      f"e2e {e2e:.4f} ms, gather ok {ok}, host == device {ok_h}", flush=True)
