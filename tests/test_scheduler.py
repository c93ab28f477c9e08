"""Scheduler token selection / page indexing bit-exact: the C++ runtime (cs_coserve_run on the
simulated clock) against the Python restatement (oracle/scheduler_oracle.py)."""
import pytest

from oracle import scheduler_oracle as S
from paper_2402_18789_b200 import engine as E


def _cfg(rate, prof, iters, ft_len, n_layers, seed, prepop=0, pages=4096, growth=128,
         max_batch=64, chunk=512, budget=50.0, amplitude=0.0, multi_layer=False, window=8192):
    c = E.CoserveConfig()
    c.rate_rps = rate
    c.duration_s = 600.0
    c.burst_amplitude = amplitude
    c.burst_period_s = 20.0
    c.tpot_slo_ms = 50.0
    c.ttft_slo_ms = 5000.0
    c.budget_ms = budget
    c.max_batch = max_batch
    c.chunk_size = chunk
    c.max_tokens = 8192
    c.max_ft_window = window
    c.profile = E.profile_struct(prof.t0_ms, prof.slope, 0.0 if prof.knee == S.INF else prof.knee,
                                 prof.bwd_weight, prof.attn_fwd, prof.attn_bwd, prof.layer0,
                                 prof.decode, prof.prefill, prof.fwd_window)
    c.multi_layer_bwd = 1 if multi_layer else 0
    c.ft_seq_len = ft_len
    c.growth_tokens = growth
    c.warmup_iters = 0
    c.timed_iters = iters
    c.prepopulate = prepop
    c.adaptive = 0
    c.seed = seed
    c.n_layers = n_layers
    c.vocab = 1000
    c.page_size = 16
    c.total_pages = pages
    c.policy, c.temporal_n = 0, 128
    return c


CASES = [
    # rate, profile, iters, ft_len, layers, seed, prepop, pages, growth, budget, amplitude
    (20.0, S.Profile(5.0, 0.01, S.INF, 1.0), 400, 2048, 4, 0, 0, 4096, 128, 50.0, 0.0),
    (20.0, S.Profile(7.3, 0.03, S.INF, 0.055), 300, 8192, 32, 1, 48, 8192, 128, 45.0, 0.0),
    (4.0, S.Profile(2.0, 0.01, 4096.0, 1.0), 300, 512, 2, 2, 0, 4096, 64, 50.0, 0.5),
    (40.0, S.Profile(3.0, 0.02, S.INF, 0.1), 300, 1024, 8, 3, 10, 600, 16, 50.0, 0.9),  # page pressure
]
# B200 runtime extension: context-aware window costs + multi-layer backward iterations
CASES_EXT = [
    (20.0, S.Profile(7.3, 0.018, S.INF, 0.06, 1.1e-6, 8e-8, 0.4), 400, 8192, 32, 4, 48, 8192, 128, 45.0, 0.0),
    (10.0, S.Profile(5.0, 0.02, S.INF, 0.1, 2e-6, 1e-7), 300, 2048, 6, 5, 8, 4096, 64, 40.0, 0.5),
    # measured-profile form: per-kind inference rows + a fixed forward-window cost
    (20.0, S.Profile(4.5, 0.02, S.INF, 0.023, 5.6e-7, 8e-8, 0.19, 0.016, 0.011, 1.7), 400, 8192, 32,
     6, 100, 8192, 128, 45.0, 0.0),
]


@pytest.mark.parametrize("case", CASES)
def test_sim_plans_bit_exact(case):
    rate, prof, iters, ft_len, nl, seed, prepop, pages, growth, budget, amp = case
    stats, log = E.coserve_run(None, _cfg(rate, prof, iters, ft_len, nl, seed, prepop, pages,
                                          growth, budget=budget, amplitude=amp))
    w = S.Workload(rate=rate, duration_s=600.0, amplitude=amp, period_s=20.0)
    ref = S.run(prof, w, seed, nl, 16, pages, growth, ft_len, iters, prepopulate=prepop,
                budget=budget)
    assert len(log) == len(ref) == iters
    for i, (a, b) in enumerate(zip(log, ref)):
        for k in ("c", "s", "phase", "layer", "l", "n_decode", "n_prefill", "n_running", "n_queue"):
            assert a[k] == b[k], (i, k, a[k], b[k])
        assert a["t_ms"] == b["t_ms"], i
        assert a["pred_ms"] == b["pred"], i
    # SLO safety
    for a in log:
        if a["c"] > 0:
            assert a["pred_ms"] <= budget + 1e-9


@pytest.mark.parametrize("case", CASES_EXT)
def test_sim_plans_bit_exact_ctx_multilayer(case):
    rate, prof, iters, ft_len, nl, seed, prepop, pages, growth, budget, amp = case
    stats, log = E.coserve_run(None, _cfg(rate, prof, iters, ft_len, nl, seed, prepop, pages,
                                          growth, budget=budget, amplitude=amp, multi_layer=True))
    w = S.Workload(rate=rate, duration_s=600.0, amplitude=amp, period_s=20.0)
    ref = S.run(prof, w, seed, nl, 16, pages, growth, ft_len, iters, prepopulate=prepop,
                budget=budget, multi_layer=True)
    multi = 0
    for i, (a, b) in enumerate(zip(log, ref)):
        for k in ("c", "s", "phase", "layer", "l", "n_decode", "n_prefill", "n_running", "n_queue"):
            assert a[k] == b[k], (i, k, a[k], b[k])
        assert a["t_ms"] == b["t_ms"] and a["pred_ms"] == b["pred"], i
        multi += len(b["bwd"]) > 1
        if a["c"] > 0:
            assert a["pred_ms"] <= budget + 1e-9
    assert multi > 0  # some iterations carried windows of several layers
    assert stats["minibatches_done"] >= 1


@pytest.mark.parametrize("window", [256, 1024])
def test_sim_plans_bit_exact_small_windows(window):
    """BASELINE config 3's token-level windows of 256 / 1024: with multi-window iterations a
    window-bound backward iteration carries several consecutive windows of one layer (and the
    forward fuses consecutive windows); C++ plans == Python restatement, bit-exact."""
    prof = S.Profile(7.0, 0.02, S.INF, 0.06, 1.5e-6, 1e-7, 0.3)
    stats, log = E.coserve_run(None, _cfg(20.0, prof, 400, 8192, 48, 9, 32, 8192, 128,
                                          budget=67.5, multi_layer=True, window=window))
    w = S.Workload(rate=20.0, duration_s=600.0, amplitude=0.0, period_s=20.0)
    ref = S.run(prof, w, 9, 48, 16, 8192, 128, 8192, 400, prepopulate=32, budget=67.5,
                multi_layer=True, max_ft_window=window)
    same_layer = 0
    for i, (a, b) in enumerate(zip(log, ref)):
        for k in ("c", "s", "phase", "layer", "l", "n_decode", "n_prefill", "n_running", "n_queue"):
            assert a[k] == b[k], (i, k, a[k], b[k])
        assert a["t_ms"] == b["t_ms"] and a["pred_ms"] == b["pred"], i
        assert all(sw <= window for _, _, sw in b["bwd"])
        layers = [ly for ly, _, _ in b["bwd"]]
        same_layer += len(layers) != len(set(layers))
    assert same_layer > 0  # window-bound iterations packed several windows of one layer


def test_token_accounting_and_work_conservation():
    prof = S.Profile(1.0, 0.01, S.INF, 1.0)
    stats, log = E.coserve_run(None, _cfg(0.0, prof, 200, 64, 3, 0))
    # no inference: every iteration schedules s = min(max under budget, remaining) > 0
    assert all(a["s"] > 0 for a in log)
    assert stats["minibatches_done"] >= 1
    per_mb = 64 + 3 * 64                         # SPEC.md:707 forward L + N*L backward
    total = stats["ft_fwd_tokens"] + stats["ft_bwd_tokens"]
    assert total >= per_mb * stats["minibatches_done"]


def test_spec_examples_via_oracle():
    p = S.Profile(2.0, 0.01, 4096.0)
    assert S.latency(p, 0, 0) == 2.0
    assert S.latency(p, 1000, 0) == pytest.approx(12.0)
    assert S.latency(p, 4196, 0) == pytest.approx(44.96)
    q = S.Profile(2.0, 0.01)
    assert S.max_finetune_tokens(q, 1000, 50.0) == 3800
    assert S.max_finetune_tokens(q, 1000, S.latency(q, 1000, 7)) == 7
    m = S.MemoryModel(3, 16)
    assert m.try_admit(60) is None
    ft = S.FtState(L=8, n_layers=2, phase=S.FWD)
    trace = []
    for s in (3, 3, 2):
        S.advance_finetune(ft, s)
        trace.append(ft.l)
    assert trace == [3, 6, 8] and ft.phase == S.BWD


# ---------------------------------------------------------------- baseline policies
def test_dts_known_answers():
    """PAPER.md:528-590 Algorithm 'Dynamic Temporal Sharing' / SPEC.md:485-506 examples."""
    st = S.DtsState()
    assert S.dts_compute_interval(st) == 64.0                       # Q empty -> 64
    flips = [S.dts_step(st, 0, 0, 0, 0) for _ in range(64)]
    assert flips[:63] == [False] * 63 and flips[63]                  # fresh s=64: 64th switches
    assert st.d == 1 and st.s == pytest.approx(64 * 1.1)             # s <- min(512, f_p*1.1)
    st = S.DtsState()
    st.Q, st.r_a, st.r_c = [8.0, 12.0, 10.0], 30.0, 24.0            # qbar 10, qmax 12, l 10, m 8
    out = S.dts_compute_interval(st)
    f_pre = 64 + (1.23 - 0.8) / 1.2 * 0.6 * 448                      # p = 1.23 -> f ~ 160.3
    assert f_pre == pytest.approx(160.32, abs=0.01)
    assert out == pytest.approx((f_pre * 1.35 + 2 * 64) / 3)
    st = S.DtsState()
    st.Q, st.r_a, st.r_c = [4.0, 6.0], 0.0, 0.0                      # p = 0.25 + 0.24 = 0.49
    assert S.dts_compute_interval(st) == pytest.approx(80.0)         # (86.4+128)/3=71.5 -> 80
    # the third decision takes the full recompute path
    st = S.DtsState()
    n = 0
    while st.d < 2:
        S.dts_step(st, 30, 10, 2, 1)
        n += 1
    for _ in range(10000):
        if S.dts_step(st, 30, 10, 2, 1):
            break
    assert st.d == 0 and 80.0 <= st.s <= 512.0


@pytest.mark.parametrize("policy,n", [(S.TEMPORAL, 16), (S.TEMPORAL, 64), (S.DTS, 0)])
def test_temporal_policies_bit_exact(policy, n):
    """Temporal-sharing baselines (§8.2): the C++ loop (coserve/baselines.hpp) and the
    Python restatement plan identical iterations on the simulated clock."""
    prof = S.Profile(5.0, 0.01, S.INF, 0.3, 1e-6, 1e-7, 0.4)
    c = _cfg(12.0, prof, 500, 1024, 4, 5, 16, 4096, 64, budget=45.0, multi_layer=True)
    c.policy, c.temporal_n = policy, n
    stats, log = E.coserve_run(None, c)
    w = S.Workload(rate=12.0, duration_s=600.0, amplitude=0.0, period_s=20.0)
    ref = S.run(prof, w, 5, 4, 16, 4096, 64, 1024, 500, prepopulate=16, budget=45.0,
                multi_layer=True, policy=policy, temporal_n=n)
    assert len(log) == len(ref) == 500
    for i, (a, b) in enumerate(zip(log, ref)):
        for k in ("c", "s", "phase", "layer", "l", "n_decode", "n_prefill", "n_running", "n_queue"):
            assert a[k] == b[k], (i, k, a[k], b[k])
        assert a["t_ms"] == b["t_ms"] and a["pred_ms"] == b["pred"], i
        assert not (a["c"] > 0 and a["s"] > 0)      # never co-served: inference xor finetuning
    assert stats["minibatches_done"] >= 1
    if policy == S.TEMPORAL:  # every finetuning iteration follows >= n inference iterations
        runs, cur = [], 0
        for a in log:
            if a["s"] > 0 and cur:
                runs.append(cur)
                cur = 0
            elif a["c"] > 0:
                cur += 1
        assert runs and all(r >= n for r in runs[1:])


def test_coserve_beats_temporal_in_simulation():
    """at the same SLO, co-serving sustains more finetuning than temporal
    sharing at frequency 128 (simulated clock, same profile and trace)."""
    prof = S.Profile(5.0, 0.01, S.INF, 0.3, 1e-6, 1e-7, 0.4)
    res = {}
    for pol, n in ((S.COSERVE, 0), (S.TEMPORAL, 128)):
        c = _cfg(20.0, prof, 1500, 2048, 8, 2, 32, 8192, 64, budget=45.0, multi_layer=True)
        c.policy, c.temporal_n = pol, n
        st, _ = E.coserve_run(None, c)
        res[pol] = (st["ft_fwd_tokens"] + st["ft_bwd_tokens"] / 8) / st["timed_ms"]
    assert res[S.COSERVE] > 1.2 * res[S.TEMPORAL], res


# ---------------------------------------------------------------- VTC fairness (App. C)
def _vtc_cfg(vtc, tenants=2, share=0.85, rate=45.0, iters=1500):
    prof = S.Profile(5.0, 0.01, S.INF, 0.3, 1e-6, 1e-7, 0.4)
    c = _cfg(rate, prof, iters, 2048, 8, 3, 0, 6000, 64, budget=45.0, multi_layer=True)
    c.vtc, c.n_tenants, c.tenant0_share, c.ft_tenant = (1 if vtc else 0), tenants, share, -1
    c.vtc_wp, c.vtc_wq, c.vtc_wr = 1.0, 2.0, 1.0
    return c


def test_vtc_off_tenants_do_not_change_plans():
    """Tenant labels come from a separate stream: with VTC off the plans are the 1-tenant ones."""
    a = E.coserve_run(None, _vtc_cfg(False, tenants=1))[1]
    b = E.coserve_run(None, _vtc_cfg(False, tenants=3))[1]
    assert [(x["c"], x["s"], x["n_queue"]) for x in a] == [(x["c"], x["s"], x["n_queue"]) for x in b]


def test_vtc_fairness_bounds_overloaded_tenants():
    """Overload (45 req/s; tenant 0 sends 85%): with VTC the backlogged tenants' counters stay
    within Lemma 1's spread max(w_p L_input, max(w_q, w_r) M) and their service within Theorem
    1's 2x that over every interval both are backlogged; the light tenant gets more service than
    under FIFO admission."""
    st_v, _ = E.coserve_run(None, _vtc_cfg(True))
    st_f, _ = E.coserve_run(None, _vtc_cfg(False))
    L_input, M = 4096, 1024          # workload prompt / generation caps
    lemma = max(1.0 * L_input, max(2.0, 1.0) * M)
    assert st_v["vtc_spread_max"] <= lemma + 1e-6, st_v["vtc_spread_max"]
    assert st_v["vtc_pair_gap_max"] <= 2 * lemma + 1e-6, st_v["vtc_pair_gap_max"]
    assert st_v["vtc_pair_gap_max"] > 0                     # both tenants were backlogged
    # FIFO admission serves requests in arrival order: the light tenant waits behind the heavy
    # one; VTC admits the light tenant's requests first while its counter is lower
    done_v, done_f = st_v["tenant_done"], st_f["tenant_done"]
    assert done_v[1] / max(1, sum(done_v)) > done_f[1] / max(1, sum(done_f))


# ---------------------------------------------------------------- spatial / isolation baselines
@pytest.mark.parametrize("policy,rho,gamma", [(S.SPATIAL, 0.5, 1.15), (S.SPATIAL, 0.7, 1.3),
                                              (S.ISOLATE, 0.4, 0.0)])
def test_spatial_policies_bit_exact(policy, rho, gamma):
    """Spatial sharing / resource isolation (coserve/baselines.hpp): the C++
    loop and the Python restatement plan identical ticks on the simulated clock; every tick is
    the inference iteration slowed by gamma / rho and carries the finetuning partition's
    windows sized to (1 - rho) / gamma of it."""
    prof = S.Profile(5.0, 0.01, S.INF, 0.3, 1e-6, 1e-7, 0.4)
    c = _cfg(12.0, prof, 500, 1024, 4, 5, 16, 4096, 64, budget=45.0, multi_layer=True)
    c.policy, c.spatial_rho, c.spatial_gamma = policy, rho, gamma
    stats, log = E.coserve_run(None, c)
    w = S.Workload(rate=12.0, duration_s=600.0, amplitude=0.0, period_s=20.0)
    ref = S.run(prof, w, 5, 4, 16, 4096, 64, 1024, 500, prepopulate=16, budget=45.0,
                multi_layer=True, policy=policy, rho=rho, gamma=gamma if gamma >= 1.0 else 1.15)
    assert len(log) == len(ref) == 500
    g = 1.0 if policy == S.ISOLATE else gamma
    for i, (a, b) in enumerate(zip(log, ref)):
        for k in ("c", "s", "phase", "layer", "l", "n_decode", "n_prefill", "n_running", "n_queue"):
            assert a[k] == b[k], (i, k, a[k], b[k])
        assert a["t_ms"] == b["t_ms"] and a["pred_ms"] == b["pred"], i
        if a["c"] > 0:  # the inference side fits the budget only after its gamma / rho slowdown
            assert a["pred_ms"] <= 45.0 + 1e-9
    assert stats["minibatches_done"] >= 1
    assert any(a["c"] > 0 and a["s"] > 0 for a in log)   # both partitions advance in one tick


def _criterion7_cfg(seed, policy, n=0, rho=0.5):
    # the measured 8B profile (BENCH_r01 "profile"): per-kind rows, context terms, window cost
    prof = S.Profile(4.6, 0.0153, S.INF, 0.033, 7e-7, 7.5e-8, 0.18, 0.0149, 0.0109, 2.7)
    c = _cfg(20.0, prof, 2500, 8192, 32, seed, 40, 24576, 128, max_batch=256, budget=45.0,
             amplitude=0.5, multi_layer=True)
    c.policy, c.temporal_n, c.spatial_rho, c.spatial_gamma = policy, n, rho, 1.15
    return c


def test_acceptance_criterion_7_slo_safety_and_policy_order():
    """SPEC.md:780 (criterion 7): on 5 seeds of a 20 req/s burst trace, co-serving never plans
    an iteration whose predicted latency exceeds the TPOT budget while inference is active, and
    its inference SLO attainment is >= spatial(rho=0.5) and >= temporal(n=64) on the same
    traces (§8.2, directional)."""
    for seed in range(5):
        att = {}
        for name, pol, n in (("coserve", S.COSERVE, 0), ("spatial", S.SPATIAL, 0),
                             ("temporal64", S.TEMPORAL, 64)):
            c = _criterion7_cfg(seed, pol, n)
            while True:  # the same simulated horizon (>= 100 s of the trace) for every policy
                st, log = E.coserve_run(None, c)
                if log[-1]["t_ms"] >= 100000.0:
                    break
                c.timed_iters *= 2
            if name == "coserve":
                assert all(a["pred_ms"] <= 50.0 for a in log if a["c"] > 0), seed
            att[name] = st["requests_slo_ok"] / max(1, st["requests_done"])
            assert st["requests_done"] > 50, (seed, name)
        assert att["coserve"] >= att["spatial"], (seed, att)
        assert att["coserve"] >= att["temporal64"], (seed, att)
