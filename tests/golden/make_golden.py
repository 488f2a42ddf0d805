"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED
reference library (oracle/_ref/libcortex_ref.so, built from /root/reference
sources by oracle/Makefile).  Run here, where /root/reference exists:

    make -C oracle all ref && python tests/golden/make_golden.py

Inputs are regenerated from cortex::Rng seeds (the Rng restatement is pinned
bit-for-bit to the reference in tests/test_oracle_pins.py), so only outputs
are stored.  Synthetic-input recipe: oracle.synthetic_group
draws keys, values, queries in that order from Rng(seed), N(0,1) fp32.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def small_cases(ref):
    """Randomised point-level cases: (seed, n, dim, k, lam, n_heads)."""
    rs = np.random.default_rng(20260118)
    cases = []
    for _ in range(60):
        n = int(rs.integers(1, 200))
        dim = int(rs.choice([1, 2, 3, 6, 8, 16, 32, 64]))
        heads = int(rs.choice([h for h in (1, 2, 4) if dim % h == 0]))
        k = int(rs.integers(1, n + 3))
        lam = float(rs.choice([0.0, 1.0, 0.5, float(rs.random())]))
        cases.append((int(rs.integers(1, 2**31)), n, dim, k, lam, heads))
    out = {"seed": [], "n": [], "dim": [], "k": [], "lam": [], "heads": [], "attn": [], "idx": [], "scores": [],
           "cov": []}
    for seed, n, dim, k, lam, heads in cases:
        r = ref.rng(seed)
        cloud = r.gaussian_f32(n * dim, 0.0, 2.0).reshape(n, dim)
        q = r.gaussian_f32(dim)
        a = ref.attention_scores_points(cloud, q, heads)
        idx, sc = ref.select_landmarks_points(cloud, a, k, lam)
        cov = ref.coverage_scores_points(cloud, idx[: max(1, len(idx) // 2)])
        for key, v in (("seed", seed), ("n", n), ("dim", dim), ("k", k), ("lam", lam), ("heads", heads)):
            out[key].append(v)
        out["attn"].append(a)
        out["idx"].append(idx)
        out["scores"].append(sc)
        out["cov"].append(cov)
    flat = {}
    for key in ("seed", "n", "dim", "k", "lam", "heads"):
        flat[key] = np.asarray(out[key])
    for key in ("attn", "idx", "scores", "cov"):
        flat[key] = np.concatenate(out[key])
        flat[key + "_off"] = np.cumsum([0] + [len(x) for x in out[key]])
    np.savez_compressed(os.path.join(HERE, "select_small.npz"), **flat)


def group_case(ref, name, seed, L, dim, n_q, k, lam, store_attn=True):
    orc = oracle.load()
    keys, values, queries = oracle.synthetic_group(orc, seed, L, dim, n_q)
    a = oracle.group_attention(ref, keys, queries)
    idx, sc = ref.select_landmarks_points(keys, a, k, lam)
    d = dict(seed=seed, L=L, dim=dim, n_q=n_q, k=k, lam=lam, idx=idx, scores=sc,
             attn_sum=np.float64(a.sum()), attn_head=a[:64].copy())
    if store_attn:
        d["attn"] = a
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)


def cfg1_cache_case(ref, seed=1):
    """cfg1 reference default path: select_landmarks(cache, q, 40, 0.5) on a
    1-layer, 1-head, d_model=64 KvCache of L=2048 context entries."""
    orc = oracle.load()
    L, dm = 2048, 64
    keys, values, queries = oracle.synthetic_group(orc, seed, L, dm, 1)
    import ctypes as C
    lib = ref.lib
    pos = np.arange(L, dtype=np.int64)
    org = np.zeros(L, np.uint8)
    k = 40
    out_src = C.c_int64(0)
    out_n = C.c_int64(0)
    opos = np.empty(k, np.int64)
    osc = np.empty(k, np.float64)
    ok = np.empty((k, dm), np.float32)
    ov = np.empty((k, dm), np.float32)
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    st = lib.ref_select_landmarks(1, 1, dm, C.c_int64(L + 1024), C.c_int64(L), P(pos, C.c_int64), P(org, C.c_uint8),
                                  P(keys, C.c_float), P(values, C.c_float), P(queries, C.c_float), k, C.c_double(0.5),
                                  C.byref(out_src), C.byref(out_n), P(opos, C.c_int64), P(osc, C.c_double),
                                  P(ok, C.c_float), P(ov, C.c_float))
    assert st == 0, st
    n = out_n.value
    np.savez_compressed(os.path.join(HERE, "cfg1_cache.npz"), seed=seed, L=L, d_model=dm, k=k, lam=0.5,
                        source_length=out_src.value, positions=opos[:n], scores=osc[:n], keys=ok[:n], values=ov[:n])


def attend_cases(ref):
    rs = np.random.default_rng(7)
    cases = []
    for _ in range(12):
        H = int(rs.choice([1, 2, 4]))
        dk = int(rs.choice([2, 8, 16, 64]))
        n = int(rs.integers(1, 260))
        seed = int(rs.integers(1, 2**31))
        cases.append((seed, n, H, dk))
    outs = []
    for seed, n, H, dk in cases:
        r = ref.rng(seed)
        dm = H * dk
        q = r.gaussian_f32(dm)
        kk = r.gaussian_f32(n * dm)
        vv = r.gaussian_f32(n * dm)
        outs.append(ref.attend(q, kk, vv, n, H, dk))
    np.savez_compressed(os.path.join(HERE, "attend.npz"), cases=np.asarray(cases, np.int64),
                        out=np.concatenate(outs), off=np.cumsum([0] + [len(o) for o in outs]))


def bench_landmarks(ref):
    import ctypes as C
    buf = C.create_string_buffer(1 << 20)
    st = ref.lib.ref_bench_landmarks(C.c_uint64(42), 100, C.c_int64(256), 16, C.c_double(0.5), buf, C.c_int64(1 << 20))
    assert st == 0
    rep = json.loads(buf.value.decode())
    with open(os.path.join(HERE, "bench_landmarks.json"), "w") as f:
        json.dump({"parameters": rep["parameters"], "verdicts": rep["verdicts"], "rows": rep["rows"][:10]}, f,
                  indent=1, sort_keys=True)


def clustered(ref):
    out = {}
    for s in range(3):
        r = ref.rng(42 + s)
        clusters = 2 + int(r.next_below(7))
        cloud, q, cl = ref.make_clustered_cloud(r, 256, 8, clusters, 6.0, 0.5)
        a = ref.attention_scores_points(cloud, q, 2)
        idx, sc = ref.select_landmarks_points(cloud, a, 16, 0.5)
        rnd = ref.random_subset(r, 256, 16)
        out[f"cloud{s}"] = cloud
        out[f"query{s}"] = q
        out[f"idx{s}"] = idx
        out[f"scores{s}"] = sc
        out[f"random{s}"] = rnd
        out[f"haus{s}"] = np.float64(ref.hausdorff_to_subset(cloud, idx))
        out[f"mpr{s}"] = np.float64(ref.mean_pairwise_reduction_subset(cloud, idx))
    np.savez_compressed(os.path.join(HERE, "clustered.npz"), **out)


def main():
    ref = oracle.load_ref()
    if ref is None:
        sys.exit("oracle/_ref/libcortex_ref.so missing: run `make -C oracle ref` (needs /root/reference)")
    small_cases(ref)
    cfg1_cache_case(ref)
    group_case(ref, "cfg1_points", seed=11, L=2048, dim=64, n_q=1, k=40, lam=0.5)
    group_case(ref, "cfg2_group", seed=1001, L=8192, dim=64, n_q=7, k=164, lam=0.5)
    group_case(ref, "cfg4_group", seed=4001, L=32768, dim=64, n_q=7, k=656, lam=0.5, store_attn=False)
    attend_cases(ref)
    bench_landmarks(ref)
    clustered(ref)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
