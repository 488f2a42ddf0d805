"""The River / Stream loop on the device (cx_cortex_*, csrc/cortex_runtime.cu;
SURVEY.md §8(f) row 2, BASELINE configs[4]) against replays of the same steps
through the single-call entry points.

Proves, on a small river model:
  * published-version semantics (SynapseBuffer::push / read_latest, synapse.hpp:115-135):
    every token's agent outputs equal a decode against exactly the synapse version the
    runtime says it read, and every published version is the exact compression of a
    context prefix the river had reached by a push point (no torn or stale buffer);
    versions are 1, 2, ... and never go backwards;
  * injection visibility (scheduler.cpp:139-156, injector.cpp:36-94): the river's logits
    at every token equal a sequential replay (encode_thought on a scratch cache, inject,
    forward_step) bit for bit, and differ from a replay without the injections.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(n_agents=9, n_layers=2, n_kv=2, d_k=64, n_q=4, L0=600, t_cap=33, vocab=256, seed=3):
    from paper_2601_01298_b200 import runtime as rt
    from paper_2601_01298_b200.model import KvCache, ModelConfig
    cfg = ModelConfig(n_layers=n_layers, n_heads=n_kv, d_model=n_kv * d_k, d_k=d_k, vocab_size=vocab,
                      max_positions=4096)
    w = rt.Weights(cfg, rt.random_flat_weights(cfg, seed))
    river = KvCache(cfg, capacity=1024)
    g = torch.Generator(device="cuda").manual_seed(seed)
    pk = torch.randn(n_layers, L0, cfg.d_model, device="cuda", generator=g)
    pv = torch.randn(n_layers, L0, cfg.d_model, device="cuda", generator=g)
    torch.cuda.synchronize()
    river.append_context_dev(pk.data_ptr(), pv.data_ptr(), 0, L0)
    torch.cuda.synchronize()
    ag = dict(
        tail_keys=torch.randn(n_agents, n_layers, n_kv, t_cap, d_k, device="cuda", generator=g),
        tail_values=torch.randn(n_agents, n_layers, n_kv, t_cap, d_k, device="cuda", generator=g),
        tail_len=torch.full((n_agents,), t_cap - 1, dtype=torch.int32, device="cuda"),
        new_keys=torch.randn(n_agents, n_layers, n_kv, d_k, device="cuda", generator=g),
        new_values=torch.randn(n_agents, n_layers, n_kv, d_k, device="cuda", generator=g),
        q=torch.randn(n_agents, n_layers, n_q, d_k, device="cuda", generator=g),
        out=torch.zeros(n_agents, n_layers, n_q, d_k, device="cuda"),
        river_queries=torch.randn(n_kv, n_layers, n_q // n_kv, d_k, device="cuda", generator=g),
    )
    return cfg, w, river, ag


def _replay_river(cfg, w, cache, river_tokens, thoughts, L0, inject_every, T, vbase, inject=True):
    """The river's steps one call at a time: (drain_injections, forward_step) per token
    -> (logits [n][vocab], final queries [n][d_model])."""
    from paper_2601_01298_b200 import runtime as rt
    from paper_2601_01298_b200.injector import inject_dev
    from paper_2601_01298_b200.model import KvCache
    logits = torch.empty(len(river_tokens), cfg.vocab_size, device="cuda")
    fq = torch.empty(len(river_tokens), cfg.d_model, device="cuda")
    for t, tok in enumerate(river_tokens):
        if inject and t % inject_every == 0:
            i = t // inject_every
            scratch = KvCache(cfg, capacity=T)  # exactly T rows: [layer][T][d]
            for j in range(T):
                rt.forward_step_dev(w, [scratch], [thoughts[i * T + j]], [vbase + i * T + j])
            torch.cuda.synchronize()
            inject_dev(cache, scratch.keys_dev(), scratch.values_dev(), vbase + i * T, T, cfg.n_layers,
                       cfg.d_model, i, L0 + t - 1, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            del scratch
        rt.forward_step_dev(w, [cache], [tok], [L0 + t], logits=logits[t], final_query=fq[t])
    torch.cuda.synchronize()
    return logits, fq


@pytest.mark.parametrize("push_mode,push_every,inject_every",
                         [("scheduler", 5, 7), ("groups", 5, 7), ("scheduler", 1, 3), ("groups", 2, 3)])
def test_cortex_versions_and_injection_visibility(push_mode, push_every, inject_every):
    from paper_2601_01298_b200 import device as cxd
    from paper_2601_01298_b200 import runtime as rt
    L0, T, k, lam, n_tok, vbase, n_steps = 600, 4, 40, 0.5, 30, 3072, 2000
    cfg, w, river, ag = _setup(L0=L0)
    replica, replica_noinj = river.clone(), river.clone()
    tk0, tv0 = ag["tail_keys"].clone(), ag["tail_values"].clone()
    rng = np.random.default_rng(11)
    river_tokens = rng.integers(0, cfg.vocab_size, n_tok).tolist()
    thoughts = rng.integers(0, cfg.vocab_size, -(-n_tok // inject_every) * T).tolist()

    cx = rt.Cortex(w, river, k=k, lam=lam, push_every=push_every, inject_every=inject_every, thought_tokens=T,
                   virtual_base=vbase, max_context=1024, push_mode=push_mode, **ag)
    hist = torch.full((n_tok + 2, 2) + cx.syn_shape, float("nan"), device="cuda")
    outh = torch.empty((n_steps,) + tuple(ag["q"].shape), device="cuda")
    logits = torch.empty(n_tok, cfg.vocab_size, device="cuda")
    stats, vers = cx.run(river_tokens, thoughts, n_steps, river_logits=logits, synapse_history=hist,
                         out_history=outh)
    torch.cuda.synchronize()
    _, _, front_ver = cx.front_synapse()

    # ---- injected rows: present, in order, and visible to the next river step
    rep, fq = _replay_river(cfg, w, replica, river_tokens, thoughts, L0, inject_every, T, vbase)
    assert np.array_equal(replica.positions(), river.positions())
    assert np.array_equal(replica.origins(), river.origins())
    for l in range(cfg.n_layers):
        assert np.array_equal(replica.layer_keys(l), river.layer_keys(l))
    assert torch.equal(rep, logits)
    noinj, _ = _replay_river(cfg, w, replica_noinj, river_tokens, thoughts, L0, inject_every, T, vbase, inject=False)
    assert not torch.equal(noinj[0], logits[0])  # the first thought lands before token 0

    # ---- published-version semantics
    assert stats["injections"] == -(-n_tok // inject_every)
    assert stats["pushes"] >= 1 and stats["last_version"] == front_ver == 1 + stats["pushes"]
    assert vers[0] == 1 and np.all(np.diff(vers.astype(np.int64)) >= 0) and vers[-1] <= front_ver
    assert len(set(vers.tolist())) >= 2, "the agent steps never overlapped a publication"
    # every published version is exactly the push of a context prefix at a push point
    ctx_rows = L0 + n_tok
    pos = river.positions()
    ctx_idx = np.nonzero(river.origins() == 0)[0]
    assert ctx_idx.size == ctx_rows and np.array_equal(pos[ctx_idx], np.arange(ctx_rows))
    d, n_kv, n_layers, dm = cfg.d_k, cfg.n_heads, cfg.n_layers, cfg.d_model
    K = torch.stack([torch.from_numpy(river.layer_keys(l).reshape(-1, dm)[ctx_idx]) for l in range(n_layers)]).cuda()
    V = torch.stack([torch.from_numpy(river.layer_values(l).reshape(-1, dm)[ctx_idx]) for l in range(n_layers)]).cuda()

    def push_of_prefix(m):
        sk = torch.empty(cx.syn_shape, device="cuda")
        sv = torch.empty(cx.syn_shape, device="cuda")
        if push_mode == "groups":
            for h in range(n_kv):
                kh, vh = K[:, :m, h * d:(h + 1) * d], V[:, :m, h * d:(h + 1) * d]
                _, _, a, b = cxd.compress_grouped(kh, vh, ag["river_queries"][h].contiguous(), k, lam)
                sk[:, h], sv[:, h] = a, b
        else:  # select_landmarks(cache, last_query): last layer, MHA with the river's final query
            q = torch.zeros(dm, device="cuda") if m == L0 else fq[m - L0 - 1]
            keys = K[n_layers - 1:, :m]
            att = cxd.attention_grouped(keys, q.reshape(1, n_kv, d).contiguous(), mode="mha")
            rows, _ = cxd.select_grouped(keys, att, k, lam)
            r = rows[0]
            sk.copy_(K[:, r].reshape(n_layers, k, n_kv, d).permute(0, 2, 1, 3))
            sv.copy_(V[:, r].reshape(n_layers, k, n_kv, d).permute(0, 2, 1, 3))
        return sk, sv

    prefixes, prev = {}, -1
    for v in range(1, front_ver + 1):
        hk, hv = hist[v, 0], hist[v, 1]
        assert not torch.isnan(hk).any(), f"version {v} was not recorded"
        found = None
        for m in range(L0 if v == 1 else prev + 1, ctx_rows + 1):
            if v > 1 and (m - L0) % push_every:
                continue
            if m not in prefixes:
                prefixes[m] = push_of_prefix(m)
            sk, sv = prefixes[m]
            if torch.equal(sk, hk) and torch.equal(sv, hv):
                found = m
                break
        assert found is not None, f"version {v} is not the push of any context prefix"
        if v == 1:
            assert found == L0
        prev = found
    # every agent step read exactly the version the runtime reports
    for v in sorted(set(vers.tolist())):
        tk, tv = tk0.clone(), tv0.clone()
        ref = torch.empty_like(ag["out"])
        cxd.decode_step(hist[v, 0].contiguous(), hist[v, 1].contiguous(), tk, tv, ag["tail_len"], ag["q"], ref,
                        ag["new_keys"], ag["new_values"])
        torch.cuda.synchronize()
        for s in np.nonzero(vers == v)[0]:
            assert torch.equal(ref, outh[s]), f"step {s}: agents' output is not the decode against version {v}"
    cx.close()


def test_cortex_create_preconditions():
    from paper_2601_01298_b200 import errors
    from paper_2601_01298_b200 import runtime as rt
    from paper_2601_01298_b200.model import Origin
    cfg, w, river, ag = _setup(n_agents=2, L0=64)
    with pytest.raises(errors.config_error):
        rt.Cortex(w, river, k=8, lam=1.5, push_every=2, inject_every=2, thought_tokens=2, virtual_base=3072,
                  max_context=128, **ag)
    with pytest.raises(errors.config_error):  # the reserved band must lie above the river
        rt.Cortex(w, river, k=8, lam=0.5, push_every=2, inject_every=2, thought_tokens=2, virtual_base=10,
                  max_context=128, **ag)
    cx = rt.Cortex(w, river, k=8, lam=0.5, push_every=2, inject_every=2, thought_tokens=2, virtual_base=3072,
                   max_context=128, **ag)
    with pytest.raises(errors.precondition_error):  # scheduler.cpp:67-74
        cx.run([1, 2, 3], [0, cfg.vocab_size, 0, 0], 4)
    cx.close()
    river.append_entry(4000, Origin.injected, np.zeros(cfg.n_layers * cfg.d_model, np.float32),
                       np.zeros(cfg.n_layers * cfg.d_model, np.float32))
    with pytest.raises(errors.precondition_error):
        rt.Cortex(w, river, k=8, lam=0.5, push_every=2, inject_every=2, thought_tokens=2, virtual_base=3072,
                  max_context=128, **ag)


def _gate_score_ref(h, t):
    """gate.cpp:27-42 in plain Python floats (fp64, sequential, no FMA)."""
    dot = na = nb = 0.0
    for a, b in zip(h.tolist(), t.tolist()):
        dot += a * b
        na += a * a
        nb += b * b
    if na == 0.0 or nb == 0.0:
        return None  # degenerate_input_error -> decide(): NaN score, rejected
    import math
    return min(1.0, max(-1.0, dot / (math.sqrt(na) * math.sqrt(nb))))


@pytest.mark.parametrize("theta", [-1.0, "median"])
def test_cortex_gate_decides_before_injection(theta):
    """The runtime with the thought gate (cfg.gate): every thought is decided
    (gate.cpp:45-61: cosine of the river's latest hidden state and the thought's last
    hidden state >= theta) before drain_injections; a rejected thought leaves the river
    cache alone and its virtual range is reused.  Checked against a host-driven replay
    (forward_step / encode / decide in Python floats / inject one call at a time): the
    gate log (scores bitwise, verdicts) and the river's logits at every token."""
    from paper_2601_01298_b200 import runtime as rt
    from paper_2601_01298_b200.injector import inject_dev
    from paper_2601_01298_b200.model import KvCache
    L0, T, k, lam, n_tok, vbase, inj = 600, 4, 40, 0.5, 24, 3072, 3
    cfg, w, river, ag = _setup(L0=L0)
    rs = np.random.default_rng(17)
    river_tokens = rs.integers(0, cfg.vocab_size, n_tok).tolist()
    thoughts = rs.integers(0, cfg.vocab_size, (n_tok // inj + 1) * T).tolist()

    def replay(cache, th):
        """-> (logits [n][vocab], gate log, injections)"""
        logits = torch.empty(n_tok, cfg.vocab_size, device="cuda")
        hid = torch.zeros(cfg.d_model, device="cuda")
        log, vnext, n_inj = [], vbase, 0
        for t, tok in enumerate(river_tokens):
            if t % inj == 0:
                i = t // inj
                scratch = KvCache(cfg, capacity=T)
                th_hid = torch.empty(cfg.d_model, device="cuda")
                for j in range(T):
                    rt.forward_step_dev(w, [scratch], [thoughts[i * T + j]], [vnext + j],
                                        hidden=th_hid if j == T - 1 else None)
                torch.cuda.synchronize()
                s = _gate_score_ref(hid.double().cpu().numpy(), th_hid.double().cpu().numpy())
                acc = s is not None and s >= th
                log.append((i, s, acc, s is None))
                if acc:
                    inject_dev(cache, scratch.keys_dev(), scratch.values_dev(), vnext, T, cfg.n_layers, cfg.d_model, i,
                               L0 + t - 1, torch.cuda.current_stream().cuda_stream)
                    torch.cuda.synchronize()
                    vnext += T
                    n_inj += 1
                del scratch
            rt.forward_step_dev(w, [cache], [tok], [L0 + t], logits=logits[t], hidden=hid)
        torch.cuda.synchronize()
        return logits, log, n_inj

    if theta == "median":  # a threshold that splits this river's thoughts
        _, log0, _ = replay(river.clone(), -1.0)
        theta = float(np.median([s for _, s, _, d in log0 if not d]))
    ref_logits, ref_log, ref_inj = replay(river.clone(), theta)
    cx = rt.Cortex(w, river, k=k, lam=lam, push_every=5, inject_every=inj, thought_tokens=T, virtual_base=vbase,
                   max_context=1024, gate=True, theta=theta, **ag)
    logits = torch.empty(n_tok, cfg.vocab_size, device="cuda")
    stats, _ = cx.run(river_tokens, thoughts, 50, river_logits=logits)
    log = cx.gate_log()
    assert len(log) == len(ref_log)
    for (i, s, a, d), (ri, rsc, ra, rd) in zip(log, ref_log):
        assert (i, a, d) == (ri, ra, rd)
        assert (np.isnan(s) and rsc is None) or s == rsc, (i, s, rsc)
    assert stats["injections"] == ref_inj == stats["thoughts_accepted"]
    assert stats["thoughts_rejected"] == len(ref_log) - ref_inj
    assert log[0][3], "the first thought meets a river without a hidden state: degenerate, rejected"
    if theta > -1.0:
        assert 0 < ref_inj < len(ref_log) - 1, "the median threshold should split the thoughts"
    assert torch.equal(logits, ref_logits), "river logits differ from the gated replay"
    cx.close()


def test_forward_step_graph_replay_matches_direct_launches():
    """forward_step on a created stream replays a captured CUDA graph (the batch is read from
    device memory); on the default stream it issues its launches directly.  Both must give
    the same bits, token after token, across a chunk-count change (every 128 rows: a new
    graph), a cache regrow (new K / V pointers inside the same graph) and a batch of two."""
    from paper_2601_01298_b200 import runtime as rt
    from paper_2601_01298_b200.model import KvCache, ModelConfig
    cfg = ModelConfig(n_layers=3, n_heads=2, d_model=128, d_k=64, vocab_size=97, max_positions=4096)
    w = rt.Weights(cfg, rt.random_flat_weights(cfg, 11))
    L0, n = 100, 70  # rows 100 .. 170: crosses 128; capacity 130 forces a regrow
    g = torch.Generator(device="cuda").manual_seed(4)
    pk = torch.randn(3, L0, 128, device="cuda", generator=g)
    pv = torch.randn(3, L0, 128, device="cuda", generator=g)

    def run(stream):
        caches = [KvCache(cfg, capacity=130), KvCache(cfg, capacity=130)]
        torch.cuda.synchronize()
        for c in caches:
            c.append_context_dev(pk.data_ptr(), pv.data_ptr(), 0, L0)
        torch.cuda.synchronize()
        logits = torch.empty(n, 2, 97, device="cuda")
        fq = torch.empty(n, 2, 128, device="cuda")
        with torch.cuda.stream(stream):
            for t in range(n):
                batch = caches if t % 3 else caches[:1]  # batches of 2 and of 1 interleaved
                rt.forward_step_dev(w, batch, [(7 * t + b) % 97 for b in range(len(batch))],
                                    [L0 + t] * len(batch), logits=logits[t, :len(batch)],
                                    final_query=fq[t, :len(batch)])
        torch.cuda.synchronize()
        for t in range(n):
            if t % 3 == 0:
                logits[t, 1] = 0.0
                fq[t, 1] = 0.0
        return logits.cpu(), fq.cpu()

    direct = run(torch.cuda.default_stream())
    graph = run(torch.cuda.Stream())
    assert torch.isfinite(direct[0]).all()
    assert torch.equal(direct[0], graph[0]) and torch.equal(direct[1], graph[1])
