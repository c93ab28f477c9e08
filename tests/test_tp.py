"""Tensor parallelism: the sharded layer math and the GPU engine's TP path.

CPU (world-size-2 gloo, the N>1 path without a GPU): each rank runs the oracle's own
forward/backward on its shard (oracle/tp_oracle.py: heads + ffn split, LoRA A row-sharded,
B replicated with the up-projection folded into the down partial sums) with
torch.distributed all-reduces at the exchange points; the result must equal the whole-model
oracle (f64, 1e-10): logits, loss, dA shards, dB, dK/dV shards, dX.

GPU (one B200): tp=2 as a single-process group -- two engines on the same device, one host
thread each, the one-shot peer all-reduce kernel -- against the oracle (same tolerances as
the tp=1 parity tests) and against the tp=1 engine.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import coserve_oracle as O
from oracle.tp_oracle import tp_shard, tp_local_arch

ARCH = O.Arch(n_layers=3, hidden=256, n_heads=4, n_kv_heads=2, head_dim=64, ffn=512,
              vocab=128, lora_rank=8, norm="rms", act="swiglu", rope=True, qkv_bias=True,
              rope_theta=10000.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tp_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def ar(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()
    W = O.init_general(ARCH, 3)
    la, Wl = tp_shard(ARCH, W, rank, world)
    toks = list(np.random.default_rng(5).integers(0, ARCH.vocab, 40))
    tr = O.forward_full(la, Wl, toks, ar=ar)
    bw = O.backward_full(la, Wl, tr, windows=[15, 25], ar=ar)
    q.put((rank, tr["logits"], tr["loss"], bw["grads"]["a"], bw["grads"]["b"],
           [bw["layers"][n]["dk"] for n in range(ARCH.n_layers)],
           [bw["layers"][n]["dv"] for n in range(ARCH.n_layers)],
           [bw["layers"][n]["dx"] for n in range(ARCH.n_layers)]))
    dist.destroy_process_group()


def test_tp_shard_shapes():
    W = O.init_general(ARCH, 3)
    la, Wl = tp_shard(ARCH, W, 1, 2)
    assert (la.n_heads, la.n_kv_heads, la.ffn) == (2, 1, 256)
    L0 = Wl["layers"][0]
    assert L0["wq"].shape == (256, 128) and L0["wk"].shape == (256, 64)
    assert L0["wo"].shape == (128, 256) and L0["w_down"].shape == (256, 256)
    assert L0["lora_a"].shape == (256, 8) and L0["lora_b"].shape == (8, 256)
    np.testing.assert_array_equal(L0["wq"], W["layers"][0]["wq"][:, 128:])
    np.testing.assert_array_equal(L0["w_down"], W["layers"][0]["w_down"][256:])
    with pytest.raises(ValueError):
        tp_local_arch(ARCH, 4)  # 2 kv heads do not split 4 ways


def test_tp2_oracle_gloo_matches_whole_model():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = O.init_general(ARCH, 3)
    toks = list(np.random.default_rng(5).integers(0, ARCH.vocab, 40))
    tr = O.forward_full(ARCH, W, toks)
    bw = O.backward_full(ARCH, W, tr, windows=[15, 25])
    tol = 1e-10
    for r in res:
        assert np.abs(r[1] - tr["logits"]).max() < tol          # replicated head
        assert abs(r[2] - tr["loss"]) < tol
    for n in range(ARCH.n_layers):
        ga = np.concatenate([res[0][3][n], res[1][3][n]], axis=0)  # A row shards
        assert np.abs(ga - bw["grads"]["a"][n]).max() < tol
        for r in res:
            assert np.abs(r[4][n] - bw["grads"]["b"][n]).max() < tol  # dB all-reduced
        if n > 0:
            dk = np.concatenate([res[0][5][n], res[1][5][n]], axis=1)  # kv-head shards
            dv = np.concatenate([res[0][6][n], res[1][6][n]], axis=1)
            assert np.abs(dk - bw["layers"][n]["dk"]).max() < tol
            assert np.abs(dv - bw["layers"][n]["dv"]).max() < tol
        for r in res:
            assert np.abs(r[7][n] - bw["layers"][n]["dx"]).max() < tol  # dX replicated


# ----------------------------------------------------------------------------------- GPU
def _plan_steps(arch, ft_tokens, fwd_windows, bwd_windows, n_inf, seed, P):
    """The same sequence of cs_step plans as tests/test_coserve_gpu.py::_run_coserve."""
    from paper_2402_18789_b200.engine import Seg, SEG_DECODE, SEG_PREFILL, SEG_FT_FWD, \
        FT_FORWARD, FT_BACKWARD
    rng = O.Rng(seed)
    free = list(range(255, -1, -1))
    take = lambda k: [free.pop() for _ in range(k)]  # noqa: E731
    L = len(ft_tokens)
    ft_pages = take((L + P - 1) // P)
    reqs = []
    for _ in range(n_inf):
        plen = rng.uniform_int(3, 20)
        toks = [rng.uniform_int(0, arch.vocab - 1) for _ in range(plen)]
        reqs.append({"tokens": toks, "pages": take((plen + 8 + P - 1) // P), "len": plen})
    steps = [("inf", [Seg(SEG_PREFILL, r["tokens"], 0, r["pages"], sample=True) for r in reqs],
              None, [(r["tokens"], 0) for r in reqs])]
    l = 0
    for s in fwd_windows:
        segs, chk = [], []
        for r in reqs:
            t = rng.uniform_int(0, arch.vocab - 1)
            segs.append(Seg(SEG_DECODE, [t], r["len"], r["pages"], sample=True))
            chk.append(([t], r["len"]))
            r["len"] += 1
        segs.append(Seg(SEG_FT_FWD, ft_tokens[l:l + s], l, ft_pages, adapter=True))
        targets = [ft_tokens[i + 1] if i + 1 < L else -1 for i in range(l, l + s)]
        steps.append(("fwd", segs, {"phase": FT_FORWARD, "seq_len": L, "l": l, "s": s,
                                    "targets": targets}, chk))
        l += s
    for n in range(arch.n_layers - 1, -1, -1):
        lj = L
        for s in bwd_windows:
            s = min(s, lj)
            steps.append(("bwd", [], {"phase": FT_BACKWARD, "seq_len": L, "l": lj, "s": s,
                                      "layer": n, "pages": ft_pages}, n))
            lj -= s
            if lj == 0:
                break
    return steps, reqs


@pytest.mark.gpu
@pytest.mark.parametrize("fused", ["1", "0"])
def test_tp2_engine_matches_oracle_and_tp1(fused, monkeypatch):
    """TP=2 as two engines on one B200 (single-process group).  fused=1: the row-parallel
    GEMMs scatter their partial tiles into the owning rank's staging slots from the epilogue
    and the owners reduce + broadcast (CS_TP_FUSED); fused=0: GEMM + one-shot all-reduce."""
    monkeypatch.setenv("CS_TP_FUSED", fused)
    from paper_2402_18789_b200.engine import Engine, TPGroup, arch_config, tp_run
    arch = ARCH
    W = O.init_general(arch, 3)
    toks = list(np.random.default_rng(5).integers(0, arch.vocab, 100))
    tr = O.forward_full(arch, W, toks)
    bw = O.backward_full(arch, W, tr)
    steps, reqs = _plan_steps(arch, toks, [40, 60], [30, 30, 40], n_inf=5, seed=7, P=16)
    cfg = arch_config(arch, page_size=16, n_pages=256, max_tokens=512, max_ft_len=100,
                      max_segments=64)
    group = TPGroup(2)
    ranks = [Engine(cfg, device=0, tp_rank=r, group=group) for r in range(2)]
    tp_run(ranks, lambda e: e.load_weights(W))
    single = Engine(cfg, device=0)
    single.load_weights(W)
    caches = [O.QkvCache(arch, r["len"] + 8) for r in reqs]
    loss_tp = loss_1 = 0.0
    diffs, diffs_1 = [], []
    kvg = {}
    for kind, segs, ft, extra in steps:
        outs = tp_run(ranks, lambda e: e.step(segs, ft=ft, want_logits=(kind != "bwd")))
        o1 = single.step(segs, ft=ft, want_logits=(kind != "bwd"))
        if kind == "bwd":
            n = extra
            if n > 0 and ft["l"] - ft["s"] == 0:  # layer done: ΔKVAccum final
                parts = tp_run(ranks, lambda e: e.kvgrad(len(toks)))
                kvg[n] = (np.concatenate([parts[0][0], parts[1][0]], axis=1),
                          np.concatenate([parts[0][1], parts[1][1]], axis=1))
            continue
        # replicated head: both ranks produce the same logits and next tokens
        np.testing.assert_array_equal(outs[0]["next_tokens"], outs[1]["next_tokens"])
        assert np.abs(outs[0]["logits"] - outs[1]["logits"]).max() == 0.0
        for i, (tk, pos) in enumerate(extra):
            lg, _ = O.forward_window(arch, W, tk, pos, caches[i], lora=False)
            diffs.append(O.scaled_err(outs[0]["logits"][i], lg[-1]))
            diffs_1.append(O.scaled_err(outs[0]["logits"][i], o1["logits"][i]))
        if kind == "fwd":
            loss_tp += outs[0]["loss_sum"]
            loss_1 += o1["loss_sum"]
    assert max(diffs) < 0.04, max(diffs)
    assert max(diffs_1) < 0.03, max(diffs_1)
    assert O.rel_err(loss_tp / 99.0, tr["loss"]) < 1e-2
    assert abs(loss_tp - loss_1) < 1e-2 * abs(loss_1)
    for l in range(arch.n_layers):
        g = tp_run(ranks, lambda e: e.lora_grads(l))
        ga = np.concatenate([g[0][0], g[1][0]], axis=0)
        gb = g[0][1] + g[1][1]  # folded LoRA: per-rank partial dB
        assert O.max_rel_err(ga, bw["grads"]["a"][l]) < 1e-2, l
        assert O.max_rel_err(gb, bw["grads"]["b"][l]) < 1e-2, l
        floor = 0.02 if l == arch.n_layers - 1 else 0.08
        assert O.scaled_err(ga, bw["grads"]["a"][l]) < floor, l
        assert O.scaled_err(gb, bw["grads"]["b"][l]) < floor, l
    for n in (1, 2):
        assert O.scaled_err(kvg[n][0], bw["layers"][n]["dk"]) < 0.08, n
        assert O.scaled_err(kvg[n][1], bw["layers"][n]["dv"]) < 0.08, n
    # Adam: dB all-reduced inside cs_adam_step -> replicated B stays identical on the ranks
    before = tp_run(ranks, lambda e: [e.lora(l) for l in range(arch.n_layers)])
    g_all = [tp_run(ranks, lambda e: e.lora_grads(l)) for l in range(arch.n_layers)]
    tp_run(ranks, lambda e: e.adam_step(1e-3))
    after = tp_run(ranks, lambda e: [e.lora(l) for l in range(arch.n_layers)])
    cfg_a = O.AdamConfig(lr=1e-3)
    for l in range(arch.n_layers):
        assert np.abs(after[0][l][1] - after[1][l][1]).max() == 0.0
        gb = g_all[l][0][1] + g_all[l][1][1]
        p = before[0][l][1].copy()
        O.adam_step(p, gb, np.zeros_like(p), np.zeros_like(p), 1, cfg_a)
        assert np.abs(after[0][l][1] - p).max() < 1e-6 + 1e-5 * np.abs(p).max()
        for r in range(2):
            pa = before[r][l][0].copy()
            O.adam_step(pa, g_all[l][r][0], np.zeros_like(pa), np.zeros_like(pa), 1, cfg_a)
            assert np.abs(after[r][l][0] - pa).max() < 1e-6 + 1e-5 * np.abs(pa).max()
    for e in ranks:
        e.close()
    single.close()
    group.close()


@pytest.mark.gpu
def test_tp2_coserve_loop_ranks_plan_identically():
    """A TP group runs the C++ co-serving loop once per rank (cs_coserve_run): the step clock
    is max-reduced over the group (cs_engine_tp_sync_max), so both ranks admit, plan, correct
    and log exactly the same iterations (no host broadcast of plans needed)."""
    from paper_2402_18789_b200.engine import (CoserveConfig, Engine, TPGroup, arch_config,
                                              coserve_run, profile_struct, tp_run)
    arch = ARCH
    cfg = arch_config(arch, page_size=16, n_pages=2048, max_tokens=1024, max_ft_len=256,
                      max_segments=80)
    group = TPGroup(2)
    ranks = [Engine(cfg, device=0, tp_rank=r, group=group) for r in range(2)]
    tp_run(ranks, lambda e: e.init_random(5))
    vals = tp_run(ranks, lambda e: e.tp_sync_max([1.0 + e.tp_rank, 7.0 - e.tp_rank]))
    assert vals[0] == vals[1] == [2.0, 7.0]
    c = CoserveConfig()
    c.rate_rps, c.duration_s, c.burst_period_s = 40.0, 600.0, 60.0
    c.tpot_slo_ms, c.ttft_slo_ms, c.budget_ms = 50.0, 5000.0, 20.0
    c.max_batch, c.chunk_size, c.max_tokens, c.max_ft_window = 32, 128, 1024, 1024
    c.profile = profile_struct(0.5, 0.002, 0.0, 0.5)
    c.multi_layer_bwd, c.ft_seq_len, c.growth_tokens = 1, 256, 32
    c.warmup_iters, c.timed_iters, c.prepopulate, c.adaptive, c.seed = 2, 60, 8, 1, 3
    res = tp_run(ranks, lambda e: coserve_run(e, c))
    (st0, log0), (st1, log1) = res
    assert len(log0) == len(log1) > 0
    keys = ("t_ms", "pred_ms", "ms", "device_ms", "c", "s", "phase", "layer", "l", "n_decode",
            "n_prefill", "n_running", "n_queue")
    for a, b in zip(log0, log1):
        assert all(a[k] == b[k] for k in keys), (a, b)
    for k in ("ft_fwd_tokens", "ft_bwd_tokens", "requests_done", "gen_tokens", "iter_p99_ms"):
        assert st0[k] == st1[k], k
    assert st0["ft_fwd_tokens"] > 0 and st0["gen_tokens"] > 0
    for e in ranks:
        e.close()
    group.close()
