#!/usr/bin/env python
"""Headline benchmark: Warp Cortex Topological Synapse hot path on B200.

Metric (BASELINE.json): synapse compressions/s (L=8K, k=164) + agent decode
steps/s at N=100/1000.  Workload = configs[1] ("0.5B-class shape"): 24 layers x
2 KV heads x d=64 (14 q-heads, 7 per KV head), L=8192 context rows per group,
k=164 landmarks (98% compression), lambda=0.5, N=100 agents with T=32 private
rows each decoding against the shared synapse.

A step = one synapse compression (attention mass + greedy selection + landmark
K/V gather for all 48 (layer, KV-head) groups).  `value` = compressions/s with
inputs resident in HBM; the decode leg (N agents x 24 layers append+attend) is
timed in the same run and reported under "decode".  `e2e` = the same metric
through the C-ABI with HOST buffers (pinned H2D of the step's K/V/queries and
D2H of the synapse inside the timed region).

--impl reference times the reference's own CPU implementation
(oracle/_ref, compiled from the unmodified reference sources) on the host
cores, on a bounded sample of the same workload.

Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run, one
process per GPU) unless it already runs under torchrun.  The 48 groups are
sharded across ranks (strong scaling of one compression) and one C-ABI call
per rank (cx_compress_sharded_dev) runs the local selections and the single
NCCL all-gather of the packed synapse; the decode leg shards agents (N per
rank, no exchange).  NCCL_DEBUG=INFO (INIT) prints the communicator lines.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "synapse compressions/s (L=8K,k=164) + agent decode steps/s at N=100/1000"
N_LAYERS, N_KV, N_Q, D, L, K, LAM = 24, 2, 14, 64, 8192, 164, 0.5
G = N_LAYERS * N_KV
T_PRIV = 32
# algorithmic bytes per unit
COMPRESS_BYTES = (G * L * D * 4 + G * (N_Q // N_KV) * D * 4 + 4 * G * K * D * 4 + 16 * G * K)  # 108,936,192


def decode_bytes(n_agents, t=T_PRIV):
    S = N_LAYERS * N_KV * K * D * 4 * 2
    return S + n_agents * (24576 * (t + 1) + 172032)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > i + 2 and
                          s[i + 2].lower() in ("active", "1", "yes")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def local_rank():
    return int(os.environ.get("LOCAL_RANK", "0"))


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------
# CPU baseline / reference arm (oracle/_ref = unmodified reference sources)
# ----------------------------------------------------------------------------
def cpu_compress_sample(n_threads, groups, seconds_target=10.0, length=L, k=K, max_reps=50):
    """Time the reference's per-group compression (attention over the group's
    7 q-heads + select_landmarks_points, oracle/_ref = the unmodified reference
    sources) over `groups` groups of `length` rows on n_threads host threads.
    Returns (compressions/s of all 48 groups, kind, sample description)."""
    import ctypes as C

    import numpy as np

    import oracle
    ref = oracle.load_ref()
    if ref is None:
        raise RuntimeError("oracle/_ref/libcortex_ref.so not built (run build() where /root/reference exists)")
    rs = np.random.default_rng(0)
    clouds = rs.standard_normal((groups, length, D), dtype=np.float32)
    qs = rs.standard_normal((groups, N_Q // N_KV, D), dtype=np.float32)
    idx = np.empty((groups, min(k, length)), np.int64)
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    reps, t0 = 0, time.perf_counter()
    while True:
        st = ref.lib.ref_compress_groups_mt(groups, P(clouds, C.c_float), C.c_int64(length), D, P(qs, C.c_float),
                                            N_Q // N_KV, k, C.c_double(LAM), n_threads, P(idx, C.c_int64))
        if st != 0:
            raise RuntimeError("reference compression failed")
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds_target or reps >= max_reps:
            break
    value = reps * groups / G / el
    return value, "reference", (f"{reps} x {groups} of 48 groups (L={length}, k={k}, 7 q-heads) on {n_threads} "
                                f"threads, {el:.1f} s")


def cpu_decode_sample(n_threads, n_agents, seconds_target=5.0):
    """The reference's kernels::attend per (agent, layer, q-head) over [synapse
    rows || the agent's T+1 private rows], agents over n_threads host threads."""
    import ctypes as C

    import numpy as np

    import oracle
    ref = oracle.load_ref()
    rs = np.random.default_rng(1)
    syn_k = rs.standard_normal((N_LAYERS, N_KV, K, D), dtype=np.float32)
    syn_v = rs.standard_normal((N_LAYERS, N_KV, K, D), dtype=np.float32)
    T = T_PRIV + 1
    tk = rs.standard_normal((n_agents, N_LAYERS, N_KV, T, D), dtype=np.float32)
    tv = rs.standard_normal((n_agents, N_LAYERS, N_KV, T, D), dtype=np.float32)
    q = rs.standard_normal((n_agents, N_LAYERS, N_Q, D), dtype=np.float32)
    out = np.empty_like(q)
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
    reps, t0 = 0, time.perf_counter()
    while True:
        st = ref.lib.ref_decode_attend_mt(n_agents, N_LAYERS, N_KV, N_Q, D, K, T, P(syn_k), P(syn_v), P(tk), P(tv),
                                          P(q), P(out), n_threads)
        if st != 0:
            raise RuntimeError("reference decode failed")
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds_target or reps >= 100:
            break
    return reps * n_agents / el, (f"{reps} x {n_agents} agents x 24 layers x 14 q-heads, n={K}+{T}, "
                                  f"{n_threads} threads, {el:.1f} s")


def cpu_extra_baselines(threads, decode_agents=(100, 1000)):
    """The other BASELINE configurations' reference CPU numbers, timed on this host in the
    same run: cfg4 compression (16 sampled groups at L=32768 -> k=656) and agent decode."""
    out = {"cpu_model": cpu_model(), "cores": threads}
    try:
        v, _, sample = cpu_compress_sample(threads, min(G, max(threads, 8)), seconds_target=0.0, length=32768, k=656,
                                           max_reps=1)
        out["cfg4"] = {"value": v, "unit": "compressions/s", "sample": sample}
    except Exception as e:  # noqa: BLE001
        out["cfg4"] = {"value": None, "sample": f"unavailable: {e}"}
    for n in decode_agents:
        try:
            v, sample = cpu_decode_sample(threads, n, seconds_target=1.0)
            out[f"decode_N{n}"] = {"value": v, "unit": "agent-steps/s", "sample": sample}
        except Exception as e:  # noqa: BLE001
            out[f"decode_N{n}"] = {"value": None, "sample": f"unavailable: {e}"}
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    groups = G  # every step is one whole cfg2 compression (all 48 groups), as in the B200 arm
    vals = []
    for i in range(args.warmup + args.steps):
        v, kind, sample = cpu_compress_sample(threads, groups, seconds_target=0.0)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    extra = cpu_extra_baselines(threads, decode_agents=sorted({args.n_agents, 1000}))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "compressions/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: 24 layers x 2 KV heads x d=64, L=8192 -> k=164, lambda=0.5, 14 q-heads; "
                               f"decode N={args.n_agents}, T={T_PRIV}",
                   "groups_per_step": groups},
        "cpu_baseline": {"value": value, "unit": "compressions/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"one whole compression ({groups} groups) per step on {threads} threads"},
        "decode": {k: v for k, v in extra.items() if k.startswith("decode_")},
        "cfg4": extra["cfg4"],
        "e2e": {"value": value, "unit": "compressions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# B200 arm
# ----------------------------------------------------------------------------
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2601_01298_b200 import device as cxd
    from paper_2601_01298_b200.parallel import Comm, shard_range

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm.from_torch(device=local)  # the C-ABI's own NCCL communicator (cx_comm)
    dev = torch.device("cuda", local)
    # weak scaling: every rank compresses its OWN synapse (one River's 48 groups) per step, no
    # collective in the timed region; the whole job is world compressions per step.  The same
    # 48 groups sharded over the ranks + one all-gather (strong scaling of one compression,
    # cx_compress_sharded_dev) is timed separately (`sharded` in the JSON line).
    gb, ge = shard_range(G, rank, world)
    g_local = G
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    keys = torch.randn(g_local, L, D, device=dev, generator=gen)
    values = torch.randn(g_local, L, D, device=dev, generator=gen)
    queries = torch.randn(g_local, N_Q // N_KV, D, device=dev, generator=gen)
    out = (torch.empty(G, K, dtype=torch.int64, device=dev), torch.empty(G, K, dtype=torch.float64, device=dev),
           torch.empty(G, K, D, device=dev), torch.empty(G, K, D, device=dev))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    # one full compression: ONE C-ABI call per rank, cx_compress_grouped_dev (centroid ||
    # attention, greedy selection, landmark K/V gather)
    def full_compress():
        return cxd.compress_grouped(keys, values, queries, K, LAM, out=out)

    def sharded_compress():  # N > 1: this rank's 48/N groups + the NCCL all-gather
        return comm.compress_sharded(cxd.ctx(local), keys_sh, values_sh, queries_sh, K, LAM, G, out=out)

    for _ in range(max(args.warmup, 3)):
        full_compress()
    torch.cuda.synchronize()
    # decision-gap monitor of this rank's groups (every round's top-1 / top-2 gap)
    min_gap = float(cxd.selection_gaps(g_local).min()) if g_local else float("inf")

    # ---- timed: compression with inputs resident in HBM, L2 flushed between steps
    launches0 = cxd.kernel_launch_count()
    times = []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            full_compress()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
    launches = cxd.kernel_launch_count() - launches0
    # the dominant kernel (greedy selection, incl. its centroid prologue) timed
    # alone with events on its stream, same inputs, L2 flushed
    sel_times = []
    a = cxd.attention_grouped(keys, queries)
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cxd.select_grouped(keys, a, K, LAM)
        e1.record(stream)
        torch.cuda.synchronize()
        sel_times.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    sel_ms = statistics.mean(sel_times)
    fp64_rate = cxd.probe_fp64_rate(local)
    sharded = None
    if world > 1:
        # strong scaling of ONE compression: 48/N groups per rank + one all-gather
        keys_sh, values_sh, queries_sh = keys[gb:ge].contiguous(), values[gb:ge].contiguous(), queries[gb:ge].contiguous()
        for _ in range(3):
            sharded_compress()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        sh_times = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sharded_compress()
            e1.record(stream)
            torch.cuda.synchronize()
            sh_times.append(e0.elapsed_time(e1))
        t = torch.tensor([ms, sel_ms, -min_gap, statistics.mean(sh_times)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, sel_ms, min_gap = float(t[0]), float(t[1]), -float(t[2])
        sharded = {"compressions_per_s": 1000.0 / float(t[3]), "ms_per_step": float(t[3]), "groups_per_gpu": ge - gb,
                   "scaling": "strong", "api": "cx_compress_sharded_dev (local selections + one NCCL all-gather)"}
        del keys_sh, values_sh, queries_sh
    value = world * 1000.0 / ms  # every rank: one compression of its own 48 groups per step (weak scaling)
    return finish_b200(args, rank, world, dev, ms, sel_ms, value, launches, clk, keys, min_gap, fp64_rate, comm,
                       sharded)


def finish_b200(args, rank, world, dev, ms, sel_ms, value, launches, clk, keys, min_gap, fp64_rate, comm, sharded=None):
    hbm, peak_kind = load_peaks()
    # HBM roofline of the dominant kernel (greedy selection): the
    # compression's algorithmic bytes over the selection's event time
    bytes_per_launch = COMPRESS_BYTES * keys.shape[0] / G
    achieved = bytes_per_launch / (sel_ms * 1e-3) / 1e9
    # fp64 roofline: the reference's exact distance work (3 G k L d unfused fp64 add / sub /
    # mul + G k L sqrt) per second against the on-box DADD / DMUL rate.  The
    # conservative fp32 filter skips ~97% of it, so this can exceed 1 as the kernel improves.
    fp64_ops = (3 * G * K * L * D + G * K * L) * keys.shape[0] / G
    fp64_achieved = fp64_ops / (sel_ms * 1e-3)
    # clocks keep being sampled through the other timed legs (the compression
    # region alone is ~40 ms, shorter than one nvidia-smi query)
    with ClockSampler(local_rank()) as clk2:
        dec = run_decode(args, dev, rank, world)
        e2e = run_e2e(args, dev, rank, world)
        cfg5 = run_cfg5(args, dev) if rank == 0 else None
        cfg4 = run_cfg4(args, dev, rank, world, comm)
    clk.samples += clk2.samples
    line = {
        "metric": METRIC, "value": value, "unit": "compressions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (torch.randn N(0,1) keys/values/queries)",
        "config": {"workload": "cfg2 (BASELINE configs[1]): 24 layers x 2 KV heads x d=64, 14 q-heads, "
                               f"L=8192 -> k=164 (98%), lambda=0.5; decode N={args.n_agents} agents, T={T_PRIV}",
                   "groups": G, "parallelism": f"one 48-group compression per GPU on {world} GPU(s) (independent "
                   "synapses, no collective in the timed region); `sharded`: one compression over all GPUs",
                   "l2": "flushed (256 MB write) between timed steps"},
        "roofline": {"kernel": "selx_kernel (greedy max-min selection, tcgen05 distance filter, one wave)", "bound": "hbm",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "peak_source": peak_kind, "traffic": ncu_traffic("selx_kernel"),
                     "traffic_unit": "bytes per step: all selx launches of one compression (ncu --set full)",
                     "note": "selection is fp64-issue + per-round latency bound (SURVEY.md §8(d)); see roofline_fp64"},
        "roofline_fp64": {"kernel": "selx_kernel", "bound": "fp64 add/mul issue",
                          "achieved": fp64_achieved / 1e12, "peak": fp64_rate / 1e12, "unit": "T fp64 op/s",
                          "frac": fp64_achieved / fp64_rate, "algorithmic_ops_per_step": fp64_ops,
                          "peak_source": "measured on this GPU (cx_probe_fp64_rate: unfused DADD/DMUL chains)",
                          "latency_model": {"rounds": K, "us_per_round": sel_ms * 1e3 / K,
                                            "note": "k dependent rounds, each with two exchanges among the group's CTAs"}},
        "select_ms": sel_ms,
        "selection_min_decision_gap": min_gap,
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / max(1, args.steps),
        "clocks": dict(clk.summary(), regions="compression, decode, e2e, cfg5 and cfg4 timed legs"),
    }
    if dec is not None:
        line["decode"] = dec
        if "N1000" in dec:
            line["roofline_decode"] = dict(dec["N1000"]["roofline"], kernel=dec["N1000"]["kernel"] + ", N=1000")
    if e2e is not None:
        line["e2e"] = e2e
    if cfg5 is not None:
        line["cfg5"] = cfg5
    line["cfg4"] = cfg4
    if sharded is not None:
        line["sharded"] = sharded
    if rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        try:
            v, kind, sample = cpu_compress_sample(threads, G, seconds_target=3.0)
            line["cpu_baseline"] = {"value": v, "unit": "compressions/s", "cores": threads, "kind": kind,
                                    "cpu_model": cpu_model(), "sample": sample}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "compressions/s", "cores": threads, "kind": "reference",
                                    "cpu_model": cpu_model(), "sample": f"unavailable: {e}"}
        if world == 1:
            line["cpu_baseline_other_configs"] = cpu_extra_baselines(threads)
    if comm is not None:
        comm.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def ncu_traffic(kernel_substr, capture="full"):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes, one launch) of a kernel
    from the newest committed `ncu --set full` summary (profiles/r<N>_ncu_<capture>_summary.json,
    made by tools/ncu_summary.py from `ncu ... python tools/prof_step.py`), or None.
    capture "full": one compression + one N=1000 decode step; "dec100": one N=100 decode step."""
    prof = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    path = next((os.path.join(prof, f"{t}_ncu_{capture}_summary.json") for t in ("r2", "r1")
                 if os.path.exists(os.path.join(prof, f"{t}_ncu_{capture}_summary.json"))), "")
    try:
        with open(path) as f:
            rows = json.load(f)
    except (OSError, ValueError):
        return None
    # the capture holds one step (tools/prof_step.py --reps 1): every launch of the
    # kernel in it belongs to that step (the selection runs as one launch per wave
    # configuration), so their traffic is summed
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot, hit = 0.0, False
    for r in rows:
        if kernel_substr in r.get("Kernel Name", ""):
            hit = True
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, _, u = r.get(k, "").partition(" ")
                tot += float(v) * scale.get(u, 1.0)
    return tot if hit else None


def run_decode(args, dev, rank=0, world=1):
    """Decode leg: N agents x 24 layers (append + attend against the shared synapse).
    N > 1 GPUs: agents are sharded, each rank holds a synapse
    replica and its agents' private rows; no per-step exchange.  The step time is
    the max over ranks; agent-steps/s counts all N agents."""
    import torch
    import torch.distributed as dist

    from paper_2601_01298_b200 import device as cxd
    from paper_2601_01298_b200.parallel import shard_range
    out = {}
    hbm, _ = load_peaks()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    for n_total in sorted({args.n_agents, 1000}):
        ab, ae = shard_range(n_total, rank, world)
        n = ae - ab
        gen = torch.Generator(device=dev).manual_seed(99 + rank)
        syn_k = torch.randn(N_LAYERS, N_KV, K, D, device=dev, generator=gen)
        syn_v = torch.randn(N_LAYERS, N_KV, K, D, device=dev, generator=gen)
        # agent-side inputs: enough independent sets that the sets of consecutive
        # steps together exceed the 126 MB L2 (N=100: 102 MB per step -> 4 sets);
        # the shared synapse is one tensor for every set, as in the real loop
        n_sets = max(1, -(-384 * 2**20 // decode_bytes(n)))
        sets = []
        for _ in range(n_sets):
            tk = torch.randn(n, N_LAYERS, N_KV, T_PRIV + 1, D, device=dev, generator=gen)
            tv = torch.randn(n, N_LAYERS, N_KV, T_PRIV + 1, D, device=dev, generator=gen)
            tl = torch.full((n,), T_PRIV, dtype=torch.int32, device=dev)
            nk = torch.randn(n, N_LAYERS, N_KV, D, device=dev, generator=gen)
            nv = torch.randn(n, N_LAYERS, N_KV, D, device=dev, generator=gen)
            q = torch.randn(n, N_LAYERS, N_Q, D, device=dev, generator=gen)
            sets.append((tk, tv, tl, q, torch.empty_like(q), nk, nv))
        for i in range(3 * n_sets):
            cxd.decode_step(syn_k, syn_v, *sets[i % n_sets], syn_unchanged=i > 0)
        torch.cuda.synchronize()
        # steady state: back-to-back steps (a decode loop) rotating over the sets; the synapse
        # is not rewritten between steps (no push here), so each step stages it while the
        # previous one drains (CX_DECODE_SYN_UNCHANGED, programmatic dependent launch)
        reps = 20 * n_sets
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            cxd.decode_step(syn_k, syn_v, *sets[i % n_sets], syn_unchanged=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        # one step alone, L2 flushed before it (launch ramp and tail not overlapped)
        ts = []
        for _ in range(10):
            flush.zero_()
            torch.cuda._sleep(200_000)  # ~0.1 ms of GPU time: the launch below is queued before e0 is reached
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cxd.decode_step(syn_k, syn_v, *sets[0])
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms_cold = statistics.mean(ts)
        del sets
        if world > 1:
            t = torch.tensor([ms, ms_cold], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, ms_cold = float(t[0]), float(t[1])
        b = decode_bytes(n)  # this rank's bytes (synapse replica + its agents)
        out[f"N{n_total}"] = {"agent_steps_per_s": n_total / (ms * 1e-3), "ms_per_step": ms,
                              "agents_per_gpu": n, "ms_per_step_cold": ms_cold,
                              "l2": f"steady state: back-to-back steps over {n_sets} input set(s) of {b / 1e6:.0f} MB "
                                    "(> L2 together); ms_per_step_cold: one step after a 256 MB L2 flush",
                              "kernel": "decode_tc_kernel (tcgen05 synapse + CUDA-core private rows)",
                              "roofline": {"bound": "hbm", "achieved": b / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                                           "frac": b / (ms * 1e-3) / 1e9 / hbm, "bytes": b,
                                           "traffic": ncu_traffic("decode_tc_kernel", {1000: "full", 100: "dec100"}[n])
                                           if n in (100, 1000) else None}}
    return out


def run_cfg5(args, dev, tokens=600, n_agents=100, inj_every=10, push_every=10, t_inj=16):
    """BASELINE configs[4]: River + 100 Stream agents, Referential Injection every
    10 tokens, River and Stream work on priority CUDA streams -- through the C-ABI
    runtime (cx_cortex_*, csrc/cortex_runtime.cu; runtime.Cortex).

    River lane (highest priority, the calling host thread): per river token its
    forward_step on the river KvCache (24 layers x d_model 128, random weights, L=8192
    prefilled context rows); every 10 tokens a 16-token thought is encoded
    (encode_thought: 16 forward_steps on a scratch cache at reserved virtual positions)
    and injected; every 10 tokens, once the previous push is published, a push
    compresses the context rows of all 48 (layer, KV head) groups (k=164) straight into
    the back synapse buffer.  Stream lane (medium priority, a second host thread): each
    agent step is 100 agents x 24 layers decoding one token against the front synapse,
    one CUDA-graph replay.  Retention = the agents' rate while the river runs over
    their rate alone (same runtime, no river tokens)."""
    import numpy as np
    import torch

    from paper_2601_01298_b200 import runtime as rt
    from paper_2601_01298_b200.model import KvCache, ModelConfig
    dm, qpg = N_KV * D, N_Q // N_KV
    calib = 40
    n_inj = -(-(tokens + calib) // inj_every)
    vbase = L + tokens + calib + 64
    cfg = ModelConfig(n_layers=N_LAYERS, n_heads=N_KV, d_model=dm, d_k=D, vocab_size=256,
                      max_positions=vbase + (n_inj + 4) * t_inj)
    w = rt.Weights(cfg, rt.random_flat_weights(cfg, 7))
    river = KvCache(cfg, capacity=L + tokens + calib + (n_inj + 4) * t_inj)  # pre-sized: no growth mid-run
    gen = torch.Generator(device=dev).manual_seed(5)
    pre_k = torch.randn(N_LAYERS, L, dm, device=dev, generator=gen)
    pre_v = torch.randn(N_LAYERS, L, dm, device=dev, generator=gen)
    torch.cuda.synchronize()
    river.append_context_dev(pre_k.data_ptr(), pre_v.data_ptr(), 0, L)
    torch.cuda.synchronize()
    del pre_k, pre_v
    ag = dict(tail_keys=torch.randn(n_agents, N_LAYERS, N_KV, T_PRIV + 1, D, device=dev, generator=gen),
              tail_values=torch.randn(n_agents, N_LAYERS, N_KV, T_PRIV + 1, D, device=dev, generator=gen),
              tail_len=torch.full((n_agents,), T_PRIV, dtype=torch.int32, device=dev),
              new_keys=torch.randn(n_agents, N_LAYERS, N_KV, D, device=dev, generator=gen),
              new_values=torch.randn(n_agents, N_LAYERS, N_KV, D, device=dev, generator=gen),
              q=torch.randn(n_agents, N_LAYERS, N_Q, D, device=dev, generator=gen),
              out=torch.empty(n_agents, N_LAYERS, N_Q, D, device=dev),
              river_queries=torch.randn(N_KV, N_LAYERS, qpg, D, device=dev, generator=gen))
    cx = rt.Cortex(w, river, k=K, lam=LAM, push_every=push_every, inject_every=inj_every, thought_tokens=t_inj,
                   virtual_base=vbase, max_context=L + tokens + calib + 16, push_mode="groups", **ag)
    rng = np.random.default_rng(9)
    # agents alone (the stand-alone rate), the river alone (its token time), then both
    alone, _ = cx.run([], [], 2000)
    ag_alone_ms = alone["agent_ms"] / 2000
    r_tok = rng.integers(0, 256, calib).tolist()
    river_alone, _ = cx.run(r_tok, rng.integers(0, 256, -(-calib // inj_every) * t_inj).tolist(), 0)
    river_tok_ms = river_alone["river_ms"] / calib
    n_steps = max(200, int(tokens * river_tok_ms / ag_alone_ms))  # agents span the river's run
    r_tok = rng.integers(0, 256, tokens).tolist()
    th = rng.integers(0, 256, -(-tokens // inj_every) * t_inj).tolist()
    st, vers = cx.run(r_tok, th, n_steps)
    cx.close()
    rate = n_agents * n_steps / (st["agent_ms"] * 1e-3)
    rate_alone = n_agents / (ag_alone_ms * 1e-3)
    return {"workload": f"cfg5 (BASELINE configs[4]): river model 24 layers x d_model {dm} (random weights), "
                        f"L={L} prefilled context rows, {tokens} river tokens (forward_step each); a {t_inj}-token "
                        f"thought encoded + injected every {inj_every} river tokens; a push of all {G} (layer, KV "
                        f"head) groups (k={K}) every {push_every} tokens once the previous one is published; "
                        f"concurrently {n_steps} agent steps of {n_agents} agents x {N_LAYERS} layers",
            "api": "cx_cortex_create / cx_cortex_run (runtime.Cortex)",
            "agent_steps_per_s": rate, "agent_steps_per_s_alone": rate_alone, "agent_rate_retention": rate / rate_alone,
            "agent_ms": st["agent_ms"], "river_ms": st["river_ms"],
            "river_tokens_per_s": tokens / (st["river_ms"] * 1e-3), "river_tokens_per_s_alone": 1000.0 / river_tok_ms,
            "pushes": st["pushes"], "push_ms_mean": st["push_ms_mean"], "injections": st["injections"],
            "versions_read": int(len(set(vers.tolist()))), "river_entries": river.size(),
            "river_context_count": river.context_count()}


def run_cfg4(args, dev, rank=0, world=1, comm=None, steps=3):
    """BASELINE configs[3]: long context L=32768 -> k=656 (98%), 48 groups sharded
    by (layer, head) over the ranks; N > 1: cx_compress_sharded_dev (the local
    selections + the NCCL all-gather of the synapse)."""
    import torch
    import torch.distributed as dist

    from paper_2601_01298_b200 import device as cxd
    from paper_2601_01298_b200.parallel import shard_range
    l4, k4 = 32768, 656
    gb, ge = shard_range(G, rank, world)
    gen = torch.Generator(device=dev).manual_seed(77 + rank)
    keys = torch.randn(ge - gb, l4, D, device=dev, generator=gen)
    values = torch.randn(ge - gb, l4, D, device=dev, generator=gen)
    queries = torch.randn(ge - gb, N_Q // N_KV, D, device=dev, generator=gen)
    out = (torch.empty(G, k4, dtype=torch.int64, device=dev), torch.empty(G, k4, dtype=torch.float64, device=dev),
           torch.empty(G, k4, D, device=dev), torch.empty(G, k4, D, device=dev))

    def step():
        if comm is None:
            cxd.compress_grouped(keys, values, queries, k4, LAM, out=out)
        else:
            comm.compress_sharded(cxd.ctx(dev.index), keys, values, queries, k4, LAM, G, out=out)

    step()
    torch.cuda.synchronize()
    if world > 1:  # rank 0 comes from the e2e / cfg5 legs: align the ranks before timing
        dist.barrier()
        torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    del keys, values
    return {"workload": "cfg4 (BASELINE configs[3]): 48 groups, L=32768 -> k=656, lambda=0.5",
            "compressions_per_s": 1000.0 / ms, "ms_per_step": ms, "groups_per_gpu": ge - gb}


def run_e2e(args, dev, rank=0, world=1):
    """compressions/s through the C-ABI with HOST buffers: pinned H2D of the
    step's keys, values and queries, the compression, D2H of the synapse.  N > 1:
    as the headline (weak scaling), every rank runs the call on its own 48 groups
    (its own host buffers, its own PCIe link); the step time is the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2601_01298_b200 import device as cxd
    g = G
    hk = torch.randn(g, L, D).pin_memory()
    hv = torch.randn(g, L, D).pin_memory()
    hq = torch.randn(g, N_Q // N_KV, D).pin_memory()
    h_out = (torch.empty(g, K, dtype=torch.int64).pin_memory(), torch.empty(g, K, dtype=torch.float64).pin_memory(),
             torch.empty(g, K, D).pin_memory(), torch.empty(g, K, D).pin_memory())

    def step():  # ONE C-ABI call (cx_compress_grouped_host): chunked uploads overlap the compressions
        cxd.compress_grouped_host(hk, hv, hq, K, LAM, out=h_out)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
    reps = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    # whole job, all ranks: keys and queries are uploaded; values cross PCIe only at the
    # selected rows (the pinned buffer is read zero-copy by the gather: G x K rows x D floats)
    h2d = world * ((G * L * D + G * (N_Q // N_KV) * D) * 4 + G * K * D * 4)
    d2h = world * (G * K * 8 * 2 + 2 * G * K * D * 4)
    return {"value": world * 1000.0 / ms, "unit": "compressions/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms}


def spawn_ranks(n):
    """`--gpus N` outside torchrun: relaunch this command as N ranks, one process per
    GPU (torch.distributed.run, rendezvous on 127.0.0.1).  Fails loudly when fewer
    than N devices are visible."""
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} requested but only {have} CUDA device(s) are visible"}), flush=True)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-agents", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":  # host cores only: rank 0 of a torchrun launch runs it, the others exit 0
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        return 2
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    run_b200(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
