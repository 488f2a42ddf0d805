"""Micro-timing of the decode step (tools only)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_01298_b200 import device as cxd
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
impls = os.environ.get("IMPLS", "tc,v2").split(",")
for impl in impls:
  cxd.set_option("decode_impl", impl)
  for N in [int(x) for x in os.environ.get("NS", "100,1000").split(",")]:
      sk = torch.randn(24, 2, 164, 64, device="cuda", generator=g); sv = torch.randn_like(sk)
      tk = torch.randn(N, 24, 2, 33, 64, device="cuda", generator=g); tv = torch.randn_like(tk)
      tl = torch.full((N,), 32, dtype=torch.int32, device="cuda")
      nk = torch.randn(N, 24, 2, 64, device="cuda", generator=g); nv = torch.randn_like(nk)
      q = torch.randn(N, 24, 14, 64, device="cuda", generator=g); o = torch.empty_like(q)
      for _ in range(3): cxd.decode_step(sk, sv, tk, tv, tl, q, o, nk, nv)
      torch.cuda.synchronize()
      e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
      e0.record()
      for _ in range(20): cxd.decode_step(sk, sv, tk, tv, tl, q, o, nk, nv, syn_unchanged=os.environ.get('PDL') == '1')
      e1.record(); torch.cuda.synchronize()
      ms = e0.elapsed_time(e1) / 20
      B = 24*2*164*64*4*2 + N*(24576*33 + 172032)
      print(f"{impl} N={N}: {ms*1000:.1f} us/step  {N/ms*1000:.0f} agent-steps/s  {B/ms/1e6:.0f} GB/s ({B/ms/1e6/6552*100:.1f}% of HBM)")
