"""Metric kernels (A7: hausdorff / mean-pairwise reduction) at scale (tools only)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.environ.get("CX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_01298_b200 as cx
for L, m in [(2048, 40), (8192, 164)]:
    rng = np.random.default_rng(0)
    cloud = rng.standard_normal((L, 64)).astype(np.float32)
    rows = np.sort(rng.choice(L, m, replace=False)).astype(np.int64)
    for name, fn in [("hausdorff_to_subset", lambda: cx.hausdorff_to_subset(cloud, rows)),
                     ("mean_pairwise_reduction_subset", lambda: cx.mean_pairwise_reduction_subset(cloud, rows))]:
        fn()
        t0 = time.perf_counter(); v = fn(); dt = time.perf_counter() - t0
        print(f"L={L} m={m} {name}: {dt*1e3:.2f} ms  ({v:.6f})", flush=True)
