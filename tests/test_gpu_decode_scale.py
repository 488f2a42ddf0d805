"""Batched decode parity at the headline sizes (BASELINE configs[1]/[2]):
24 layers x 2 KV heads x 14 q-heads, d_k = 64, k_syn = 164, t_cap = 33, at
N = 1000 and N = 2000 agents -- EVERY agent, layer and q-head checked against
the oracle (kernels.cpp:103-142 attend with n_heads = 1 over [synapse rows ||
private rows], scheduler.cpp:245-262).

At N = 1000 the launch is 48 (layer, KV head) x 3 CTAs, each looping over
~19 tiles of 18 agents (N = 2000: ~37 tiles): the cross-tile pipelined S / P.V
chain, the parity-split mbarriers and the epilogue counter run through many
phases here, which the small parity cases (<= 2 tiles per CTA) never reach.

The bar (north_star "1e-3 relative, fp32 accumulate"), per output row o of one
(agent, layer, q-head) against the oracle row e:
    max_c |o_c - e_c| <= DECODE_RTOL * max_c |e_c|
i.e. relative to the row's magnitude (an attention output is a convex
combination of value rows, so near-zero coordinates carry the row's absolute
error, not a relative one).  The measured worst ratios are printed.  A
negative control (test_negative_control_bf16_only_scores) runs the same
check on a test-only build whose score GEMM drops the bf16 lo terms and
requires it to FAIL the bar: the bar is tight enough to see that regression.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DECODE_RTOL = 1e-3
N_LAYERS, N_KV, N_Q, DK, KSYN, TCAP = 24, 2, 14, 64, 164, 33
NEGCTL_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "negctl", "libcortex_negctl.so")


def _inputs(n, seed, qscale=1.0):
    import torch
    gen = torch.Generator(device="cuda").manual_seed(seed)
    syn_k = torch.randn(N_LAYERS, N_KV, KSYN, DK, device="cuda", generator=gen)
    syn_v = torch.randn(N_LAYERS, N_KV, KSYN, DK, device="cuda", generator=gen)
    tk = torch.randn(n, N_LAYERS, N_KV, TCAP, DK, device="cuda", generator=gen)
    tv = torch.randn(n, N_LAYERS, N_KV, TCAP, DK, device="cuda", generator=gen)
    # ragged tails: 0 .. t_cap - 1 stored rows (the appended row makes 1 .. t_cap)
    tl = torch.randint(0, TCAP, (n,), device="cuda", generator=gen).to(torch.int32)
    tl[:3] = torch.tensor([0, TCAP - 1, TCAP // 2], dtype=torch.int32)
    nk = torch.randn(n, N_LAYERS, N_KV, DK, device="cuda", generator=gen)
    nv = torch.randn(n, N_LAYERS, N_KV, DK, device="cuda", generator=gen)
    q = torch.randn(n, N_LAYERS, N_Q, DK, device="cuda", generator=gen) * qscale
    return syn_k, syn_v, tk, tv, tl, nk, nv, q


def row_errors(o, e):
    """(worst row ratio max|o-e| / max|e|, worst abs error, worst unit-floor ratio)."""
    d = np.abs(o.astype(np.float64) - e.astype(np.float64))
    row_err = d.max(axis=-1)
    row_mag = np.abs(e.astype(np.float64)).max(axis=-1)
    ratio = row_err / np.maximum(row_mag, 1e-30)
    unit = (d / np.maximum(1.0, np.abs(e))).max()
    return float(ratio.max()), float(d.max()), float(unit)


def _check_all(orc, syn_k, syn_v, tk0, tv0, tl, nk, nv, q, out, tk, tv):
    """Appended rows bitwise, untouched rows bitwise, every output row vs the oracle."""
    tln = tl.cpu().numpy()
    tkn, tvn = tk.cpu().numpy(), tv.cpu().numpy()
    nkn, nvn = nk.cpu().numpy(), nv.cpu().numpy()
    a = np.arange(len(tln))
    assert np.array_equal(tkn[a, :, :, tln], nkn) and np.array_equal(tvn[a, :, :, tln], nvn)
    # rows other than the appended one are untouched
    mask = np.ones(tkn.shape[:4], bool)
    mask[a, :, :, tln] = False
    assert np.array_equal(tkn[mask], tk0[mask]) and np.array_equal(tvn[mask], tv0[mask])
    exp = orc.decode_attend(syn_k.cpu().numpy(), syn_v.cpu().numpy(), tkn, tvn, tln + 1, q.cpu().numpy())
    return row_errors(out.cpu().numpy(), exp)


@pytest.mark.parametrize("n", [1000, 2000])
def test_decode_headline_every_agent(orc, n):
    import torch

    from paper_2601_01298_b200 import device
    torch.cuda.set_device(0)
    syn_k, syn_v, tk, tv, tl, nk, nv, q = _inputs(n, 100 + n)
    tk0, tv0 = tk.cpu().numpy(), tv.cpu().numpy()
    out = torch.full_like(q, float("nan"))
    device.decode_step(syn_k, syn_v, tk, tv, tl, q, out, nk, nv)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out).all()), "rows left unwritten"
    ratio, worst_abs, unit = _check_all(orc, syn_k, syn_v, tk0, tv0, tl, nk, nv, q, out, tk, tv)
    print(f"\n[decode N={n}] worst row-relative error {ratio:.3e} (bar {DECODE_RTOL:g}), "
          f"worst abs {worst_abs:.3e}, worst unit-floor {unit:.3e}")
    assert ratio <= DECODE_RTOL, ratio


def test_decode_sharp_softmax(orc):
    """q scaled x4: peaked softmax rows (the synapse / private merge with very
    different maxima), N = 1000."""
    import torch

    from paper_2601_01298_b200 import device
    syn_k, syn_v, tk, tv, tl, nk, nv, q = _inputs(1000, 7, qscale=4.0)
    tk0, tv0 = tk.cpu().numpy(), tv.cpu().numpy()
    out = torch.full_like(q, float("nan"))
    device.decode_step(syn_k, syn_v, tk, tv, tl, q, out, nk, nv)
    torch.cuda.synchronize()
    ratio, worst_abs, unit = _check_all(orc, syn_k, syn_v, tk0, tv0, tl, nk, nv, q, out, tk, tv)
    print(f"\n[decode N=1000 q x4] worst row-relative error {ratio:.3e}, worst abs {worst_abs:.3e}")
    assert ratio <= DECODE_RTOL, ratio


def _negctl_decode(syn_k, syn_v, tk, tv, tl, q, out, nk, nv):
    import torch

    from paper_2601_01298_b200._lib import CxDecodeBatch
    lib = C.CDLL(NEGCTL_SO)
    ctx = C.c_void_p()
    assert lib.cx_ctx_create(0, C.byref(ctx)) == 0
    b = CxDecodeBatch()
    n_layers, n_kv, k_syn, d_k = syn_k.shape
    b.n_agents, b.n_layers, b.n_kv, b.n_q, b.d_k, b.k_syn = q.shape[0], n_layers, n_kv, q.shape[2], d_k, k_syn
    b.syn_keys, b.syn_values = syn_k.data_ptr(), syn_v.data_ptr()
    b.tail_keys, b.tail_values, b.t_cap, b.tail_len = tk.data_ptr(), tv.data_ptr(), tk.shape[3], tl.data_ptr()
    b.new_keys, b.new_values, b.q, b.out = nk.data_ptr(), nv.data_ptr(), q.data_ptr(), out.data_ptr()
    lib.cx_decode_step_dev.argtypes = [C.c_void_p, C.POINTER(CxDecodeBatch), C.c_void_p]
    st = lib.cx_decode_step_dev(ctx, C.byref(b), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    lib.cx_ctx_destroy.argtypes = [C.c_void_p]
    lib.cx_ctx_destroy(ctx)
    assert st == 0


def test_negative_control_bf16_only_scores(orc):
    """Test-only build (tests/negctl, -DCX_NEGCTL_BF16_S): S = Q_hi K_hi only.
    The same check must FAIL on it, and pass on the product library."""
    import torch

    from paper_2601_01298_b200 import device
    if not os.path.exists(NEGCTL_SO):
        pytest.fail(f"{NEGCTL_SO} not built (run __graft_entry__.build())")
    syn_k, syn_v, tk, tv, tl, nk, nv, q = _inputs(200, 21)
    tk0, tv0 = tk.cpu().numpy(), tv.cpu().numpy()
    res = {}
    for name in ("product", "negctl"):
        tkx, tvx = tk.clone(), tv.clone()
        out = torch.full_like(q, float("nan"))
        if name == "product":
            device.decode_step(syn_k, syn_v, tkx, tvx, tl, q, out, nk, nv)
        else:
            _negctl_decode(syn_k, syn_v, tkx, tvx, tl, q, out, nk, nv)
        torch.cuda.synchronize()
        res[name] = _check_all(orc, syn_k, syn_v, tk0, tv0, tl, nk, nv, q, out, tkx, tvx)
    print(f"\n[negative control] product worst row-relative {res['product'][0]:.3e}, "
          f"bf16-only S {res['negctl'][0]:.3e} (bar {DECODE_RTOL:g})")
    assert res["product"][0] <= DECODE_RTOL
    assert res["negctl"][0] > DECODE_RTOL, "the bar does not detect a bf16-only score GEMM"
