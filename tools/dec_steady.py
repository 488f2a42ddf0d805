"""Decode steady state as bench.py measures it (tools only): back-to-back steps over enough
input sets to exceed L2, PDL with an unchanged synapse.  NS=100,1000; CX_TC_SKIP / CX_TC_TRACE
need an experiments build (tools/build_variant.sh exp WORKTREE -DCX_EXPERIMENTS)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
if os.environ.get("PER_LH"):
    cxd.set_option("decode_ctas_per_lh", int(os.environ["PER_LH"]))
tag = os.environ.get("TAG", "")
for N in [int(x) for x in os.environ.get("NS", "100,1000").split(",")]:
    B = 24 * 2 * 164 * 64 * 4 * 2 + N * (24576 * 33 + 172032)
    n_sets = max(1, -(-384 * 2**20 // B))
    sk = torch.randn(24, 2, 164, 64, device="cuda", generator=g); sv = torch.randn_like(sk)
    sets = []
    for _ in range(n_sets):
        tk = torch.randn(N, 24, 2, 33, 64, device="cuda", generator=g); tv = torch.randn_like(tk)
        tl = torch.full((N,), 32, dtype=torch.int32, device="cuda")
        nk = torch.randn(N, 24, 2, 64, device="cuda", generator=g); nv = torch.randn_like(nk)
        q = torch.randn(N, 24, 14, 64, device="cuda", generator=g); o = torch.empty_like(q)
        sets.append((tk, tv, tl, q, o, nk, nv))
    for i in range(3 * n_sets):
        cxd.decode_step(sk, sv, *sets[i % n_sets], syn_unchanged=i > 0)
    torch.cuda.synchronize()
    reps = 20 * n_sets
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record()
        for i in range(reps):
            cxd.decode_step(sk, sv, *sets[i % n_sets], syn_unchanged=True)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    print(f"{tag} N={N}: {best*1000:.1f} us/step  {B/best/1e6/6553*100:.1f}% of HBM", flush=True)
    if os.environ.get("TRACE_ONE"):
        os.environ["CX_TC_TRACE"] = "1"
        cxd.decode_step(sk, sv, *sets[0], syn_unchanged=True)
        torch.cuda.synchronize()
        del os.environ["CX_TC_TRACE"]
