"""Tensor-core selection (select_tc.cu) vs the CUDA-core kernels: bitwise agreement
on a few shapes, then cfg2 / cfg4 timings of both (tools only)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd  # noqa: E402

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)


def run(keys, a, k, impl, flags=0):
    cxd.set_option("select_impl", impl)
    r = cxd.select_grouped(keys, a, k, 0.5, flags)
    torch.cuda.synchronize()
    return r


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


shapes = [(3, 3000, 61), (2, 5, 9), (1, 2048, 40), (4, 300, 300), (5, 8192, 164)]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    shapes = shapes[:1]
for G, L, k in shapes:
    keys = torch.randn(G, L, 64, device="cuda", generator=g)
    q = torch.randn(G, 7, 64, device="cuda", generator=g)
    a = cxd.attention_grouped(keys, q)
    r_tc = run(keys, a, k, "tc")
    r_cc = run(keys, a, k, "cuda_core")
    same = torch.equal(r_tc[0], r_cc[0]) and torch.equal(r_tc[1], r_cc[1])
    print(f"G={G} L={L} k={k}: tc == cuda_core: {same}", flush=True)
for G, L, k in [(48, 8192, 164), (48, 32768, 656)]:
    keys = torch.randn(G, L, 64, device="cuda", generator=g)
    q = torch.randn(G, 7, 64, device="cuda", generator=g)
    a = cxd.attention_grouped(keys, q)
    r_tc = run(keys, a, k, "tc")
    r_cc = run(keys, a, k, "cuda_core")
    same = torch.equal(r_tc[0], r_cc[0]) and torch.equal(r_tc[1], r_cc[1])
    t_tc = timeit(lambda: run(keys, a, k, "tc"))
    for C in (3, 4, 5, 6):
        cxd.set_option("select_cluster", C)
        print(f"   forced C={C}: {timeit(lambda: run(keys, a, k, 'tc')):.3f} ms", flush=True)
    cxd.set_option("select_cluster", 0)
    t_cc = timeit(lambda: run(keys, a, k, "cuda_core"))
    print(f"G={G} L={L} k={k}: same={same}  tc {t_tc:.3f} ms  cuda_core {t_cc:.3f} ms", flush=True)
    del keys
