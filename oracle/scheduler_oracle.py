"""oracle/scheduler_oracle.py -- TEST INFRASTRUCTURE ONLY.

Pure-Python restatement of the spec-only host modules the reference defines but never
implemented:

  * latency / max_finetune_tokens / MemoryModel.try_admit
  * plan_iteration / advance_finetune / enforce_dependencies
  * generate_trace (sinusoidal Poisson thinning, lognormal)
  * run (discrete-event loop, simulated clock)

It mirrors the C++ runtime (include/coserve/*.hpp) decision for decision so the tests can
demand bit-exact plans (token selection, page ids) from cs_coserve_run(engine=NULL).
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field
from typing import List, Optional

from .coserve_oracle import Rng

INF = float("inf")


@dataclass
class Profile:
    t0_ms: float = 2.0
    slope: float = 0.01
    knee: float = INF
    bwd_weight: float = 1.0
    attn_fwd: float = 0.0   # B200 runtime extension: context term of a forward window
    attn_bwd: float = 0.0   # ... of a backward window
    layer0: float = 1.0     # cost factor of a (pruned) layer-0 backward window
    decode: float = 0.0     # per-decode-row slope of the inference rows (0 = slope)
    prefill: float = 0.0    # per-prefill-token slope (0 = slope)
    fwd_window: float = 0.0  # fixed cost of a finetuning forward window (0 = none)

    def has_ctx(self):
        return self.attn_fwd > 0 or self.attn_bwd > 0

    def has_rows(self):
        return self.decode > 0 or self.prefill > 0


def inference_cost(p: "Profile", n_dec: int, n_pre: int) -> float:
    """coserve::inference_cost (include/coserve/cost_model.hpp)."""
    if not p.has_rows():
        return latency(p, n_dec + n_pre, 0)
    d = p.decode if p.decode > 0 else p.slope
    f = p.prefill if p.prefill > 0 else p.slope
    return p.t0_ms + d * float(n_dec) + f * float(n_pre)


def ft_fwd_cost(p: Profile, l: int, s: int) -> float:
    return ((p.fwd_window if s > 0 else 0.0) + p.slope * float(s)
            + p.attn_fwd * float(s) * (float(l) + 0.5 * float(s)))


def ft_bwd_cost(p: Profile, lj: int, s: int, layer: int = 1) -> float:
    w = p.bwd_weight if p.bwd_weight > 0 else 1.0
    c = w * p.slope * float(s) + p.attn_bwd * float(s) * (float(lj) - 0.5 * float(s))
    return p.layer0 * c if layer == 0 else c


def max_tokens_within(cost, cap: int, room: float) -> int:
    if cap <= 0 or room <= 0 or cost(1) > room:
        return 0
    lo, hi = 1, cap
    while lo < hi:
        mid = lo + (hi - lo + 1) // 2
        if cost(mid) <= room:
            lo = mid
        else:
            hi = mid - 1
    return lo


def latency(p: Profile, c: int, s: int) -> float:
    """SPEC.md:353-361."""
    if c < 0 or s < 0:
        raise ValueError("latency: c, s must be >= 0")
    n = float(c) + float(s)
    return p.t0_ms + p.slope * min(n, p.knee) + 2.0 * p.slope * max(0.0, n - p.knee)


def max_finetune_tokens(p: Profile, c: int, budget: float) -> int:
    """largest s with latency(c, s) <= budget (inclusive); 0 if none."""
    if not budget > 0:
        raise ValueError("budget must be > 0")
    if latency(p, c, 0) > budget:
        return 0
    b, k = p.slope, p.knee
    rem = budget - p.t0_ms
    if b <= 0:
        return 2 ** 31 - 1
    n = rem / b if rem / b <= k else k + (rem - b * k) / (2.0 * b)
    s = max(0, int(math.floor(n)) - c)
    while s > 0 and latency(p, c, s) > budget:
        s -= 1
    while latency(p, c, s + 1) <= budget:
        s += 1
    return s


class MemoryModel:
    """SPEC.md:346-351,371-379 with a LIFO free list (deterministic page ids)."""

    def __init__(self, total_pages: int, page_size: int, growth_tokens: int = 0):
        self.page = page_size
        self.growth = growth_tokens
        self.free = list(range(total_pages - 1, -1, -1))

    def pages_for(self, tokens: int) -> int:
        return (tokens + self.page - 1) // self.page

    def try_admit(self, prompt: int):
        need = self.pages_for(prompt) + self.pages_for(self.growth)
        if need > len(self.free) or prompt < 0:
            return None
        return [self.free.pop() for _ in range(need)]

    def reserve(self, n: int):
        if n > len(self.free):
            return None
        return [self.free.pop() for _ in range(n)]

    def grow(self, pages: List[int]) -> bool:
        if not self.free:
            return False
        pages.append(self.free.pop())
        return True

    def release(self, pages: List[int]):
        for p in reversed(pages):
            self.free.append(p)


class TraceRng:
    """workload.hpp TraceRng == rng.hpp distributions over mt19937_64."""

    def __init__(self, seed):
        self.r = Rng(seed)

    def uniform(self):
        return self.r.uniform()

    def uniform_int(self, lo, hi):
        return self.r.uniform_int(lo, hi)

    def lognormal(self, mu, sigma):
        return self.r.lognormal(mu, sigma)

    def exponential(self, rate):
        return self.r.exponential(rate)


def clip_len(v: float, lo: int, hi: int) -> int:
    r = int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))  # std::lround
    return max(lo, min(hi, r))


@dataclass
class Workload:
    rate: float = 20.0
    duration_s: float = 60.0
    amplitude: float = 0.0
    period_s: float = 60.0
    prompt_mu: float = 5.5
    prompt_sigma: float = 0.8
    prompt_min: int = 16
    prompt_max: int = 4096
    gen_mu: float = 4.5
    gen_sigma: float = 0.7
    gen_min: int = 8
    gen_max: int = 1024


def generate_trace(w: Workload, seed: int):
    """SPEC.md:635-643 (draw order per candidate: gap, accept; per arrival: prompt, gen)."""
    if w.amplitude < 0 or w.amplitude > 1:
        raise ValueError("amplitude must be in [0, 1]")
    out = []
    if w.rate <= 0 or w.duration_s <= 0:
        return out
    rng = TraceRng(seed)
    lam_max = w.rate * (1.0 + w.amplitude)
    t = 0.0
    while True:
        t += rng.exponential(lam_max)
        if t >= w.duration_s:
            break
        lam = w.rate * (1.0 + w.amplitude * math.sin(2.0 * math.pi * t / w.period_s))
        u = rng.uniform()
        if u * lam_max > lam:
            continue
        p = clip_len(rng.lognormal(w.prompt_mu, w.prompt_sigma), w.prompt_min, w.prompt_max)
        g = clip_len(rng.lognormal(w.gen_mu, w.gen_sigma), w.gen_min, w.gen_max)
        out.append((t * 1000.0, p, g))
    return out


@dataclass
class Request:
    id: int
    prompt_len: int
    gen_len: int
    arrival_ms: float
    prefilled: int = 0
    emitted: int = 0
    pages: List[int] = field(default_factory=list)
    first_token_ms: float = -1.0
    completion_ms: float = -1.0

    def done(self):
        return self.emitted >= self.gen_len

    def in_prefill(self):
        return self.prefilled < self.prompt_len

    def context(self):
        return self.prefilled + max(0, self.emitted - 1)


FWD, BWD, DONE = 1, 2, 3


@dataclass
class FtState:
    L: int
    n_layers: int
    phase: int = 0
    minibatch: int = -1
    l: int = 0
    layer: int = 0
    lj: int = 0


def advance_finetune(ft: FtState, s: int):
    """SPEC.md:430-438."""
    if s <= 0:
        return
    if ft.phase == FWD:
        s = min(s, ft.L - ft.l)
        ft.l += s
        if ft.l >= ft.L:
            ft.phase, ft.layer, ft.lj = BWD, ft.n_layers - 1, ft.L
    elif ft.phase == BWD:
        s = min(s, ft.lj)
        ft.lj -= s
        if ft.lj == 0:
            ft.layer -= 1
            ft.lj = ft.L
            if ft.layer < 0:
                ft.phase = DONE


def plan_iteration(queue: deque, running: List[Request], ft: FtState, prof: Profile,
                   max_batch: int, chunk: int, max_tokens: int, max_ft_window: int,
                   mem: MemoryModel, budget: float, multi_layer: bool = False):
    """SPEC.md:421-429.  Returns a dict mirroring coserve::IterationPlan."""
    while queue and len(running) < max_batch:
        r = queue[0]
        pages = mem.try_admit(r.prompt_len)
        if pages is None:
            break
        r.pages = pages
        running.append(r)
        queue.popleft()
    def fits(nd, np_):
        return nd + np_ <= max_tokens and inference_cost(prof, nd, np_) <= budget

    n_dec = n_pre = 0
    decode, prefill = [], []
    for i, r in enumerate(running):
        if not r.in_prefill() and not r.done() and fits(n_dec + 1, 0):
            decode.append(i)
            n_dec += 1
    for i, r in enumerate(running):
        if not r.in_prefill():
            continue
        room = max_tokens_within(lambda x: 0.0 if fits(n_dec, n_pre + x) else 1.0,
                                 max_tokens - n_dec - n_pre, 0.5)
        if room <= 0:
            break
        ln = min(chunk, r.prompt_len - r.prefilled, room)
        if ln <= 0:
            continue
        prefill.append((i, r.prefilled, ln))
        n_pre += ln
    c = n_dec + n_pre
    w_b = prof.bwd_weight if prof.bwd_weight > 0 else 1.0
    s, phase, layer, l = 0, 0, -1, 0
    bwd = []
    if not prof.has_ctx() and not multi_layer:
        if ft.phase in (FWD, BWD):
            s = max_finetune_tokens(prof, c, budget)
            if ft.phase == BWD and w_b != 1.0:
                s = int(math.floor(s / w_b))
            s = min(s, (ft.L - ft.l) if ft.phase == FWD else ft.lj)
            s = min(s, max_ft_window)
            s = min(s, (max_tokens - c) if ft.phase == FWD else max_tokens)
            s = max(s, 0)
            if s > 0:
                phase = ft.phase
                layer = ft.layer if ft.phase == BWD else -1
                l = ft.l if ft.phase == FWD else ft.lj
                if ft.phase == BWD:
                    bwd.append((ft.layer, ft.lj, s))
        s_eq = int(math.ceil(s * w_b)) if (phase == BWD and w_b != 1.0) else s
        pred = latency(prof, c, s_eq)
    else:
        base = inference_cost(prof, len(decode), c - len(decode))
        room = budget - base
        cost = 0.0
        if ft.phase == FWD:
            # multi-window iterations: consecutive forward windows fuse into one segment
            # (Alg. 2 windows are additive), so the window cap does not bind
            cap = min(ft.L - ft.l, max_tokens - c) if multi_layer else \
                min(ft.L - ft.l, max_ft_window, max_tokens - c)
            l0 = ft.l
            s = max_tokens_within(lambda x: ft_fwd_cost(prof, l0, x), cap, room)
            if s > 0:
                phase, l = FWD, ft.l
                cost = ft_fwd_cost(prof, l0, s)
        elif ft.phase == BWD:
            ly, lj = ft.layer, ft.lj
            while ly >= 0 and room > 0:
                cap = min(lj, max_ft_window, max_tokens)
                sw = max_tokens_within(lambda x, lj0=lj, ly0=ly: ft_bwd_cost(prof, lj0, x, ly0),
                                       cap, room)
                if sw <= 0:
                    break
                cw = ft_bwd_cost(prof, lj, sw, ly)
                bwd.append((ly, lj, sw))
                s += sw
                cost += cw
                room -= cw
                lj -= sw
                if not multi_layer:
                    break
                if lj > 0:
                    if sw < cap:   # budget-bound: the iteration is full
                        break
                    continue       # window-bound: the next window of the same layer
                ly -= 1
                lj = ft.L
            if bwd:
                phase, layer, l = BWD, bwd[0][0], bwd[0][1]
        pred = base + cost
    return {"decode": decode, "prefill": prefill, "c": c, "s": s, "phase": phase,
            "layer": layer, "l": l, "pred": pred, "bwd": bwd}


# ---------------------------------------------------------------- baseline policies
# PAPER.md §8.2 / SPEC.md:474-548 (include/coserve/baselines.hpp)
COSERVE, TEMPORAL, DTS, SPATIAL, ISOLATE = 0, 1, 2, 3, 4


class DtsState:
    """PAPER.md:536-541 state; f_p starts at 64 (SPEC.md design decision)."""

    def __init__(self):
        self.Q, self.B = [], []
        self.r_a = self.r_c = 0.0
        self.s = 64.0
        self.f_p = 64.0
        self.d = 0


def dts_compute_interval(st: DtsState) -> float:
    """Compute_Next_Interval."""
    if not st.Q:
        return 64.0
    n = float(len(st.Q))
    qbar = sum(st.Q) / n
    qmax = max(st.Q)
    lam, mu = st.r_a / n, st.r_c / n
    p = min(1.0, qbar / 20.0) + min(0.5, qmax / 25.0) + max(0.0, (lam - mu) / 8.0)
    if p <= 0.8:
        f = 64.0
    elif p >= 2.0:
        f = 512.0
    else:
        f = 64.0 + (p - 0.8) / 1.2 * 0.6 * (512.0 - 64.0)
    f *= 1.35
    fs = (f + 2.0 * st.f_p) / 3.0
    st.f_p = fs
    fs = max(fs, 64.0 + 16.0)
    return min(512.0, max(64.0, fs))


def dts_step(st: DtsState, q, b, a, c) -> bool:
    """Scheduler_Step: True = switch to finetuning."""
    st.r_a += a
    st.r_c += c
    st.Q.append(float(q))
    st.B.append(float(b))
    st.s -= 1.0
    if st.s <= 0.0:
        st.d += 1
        if st.d >= 3:
            st.s = dts_compute_interval(st)
            st.d = 0
        else:
            st.s = min(512.0, st.f_p * 1.1)
        st.Q, st.B, st.r_a, st.r_c = [], [], 0.0, 0.0
        return True
    return False


def plan_ft_block(ft: "FtState", prof: Profile, max_tokens: int, max_ft_window: int):
    """One step of a temporal-sharing finetuning iteration (baselines.hpp plan_ft_block)."""
    pred = inference_cost(prof, 0, 0)
    s, phase, layer, l, bwd = 0, 0, -1, 0, []
    if ft.phase == FWD:
        s = min(ft.L - ft.l, max_tokens)
        if s > 0:
            phase, l = FWD, ft.l
            pred += ft_fwd_cost(prof, ft.l, s)
    elif ft.phase == BWD:
        s = min(ft.lj, max_ft_window, max_tokens)
        if s > 0:
            phase, layer, l = BWD, ft.layer, ft.lj
            bwd = [(ft.layer, ft.lj, s)]
            pred += ft_bwd_cost(prof, ft.lj, s, ft.layer)
    return {"decode": [], "prefill": [], "c": 0, "s": s, "phase": phase, "layer": layer,
            "l": l, "pred": pred, "bwd": bwd}


def run(prof: Profile, w: Workload, seed: int, n_layers: int, page_size: int, total_pages: int,
        growth: int, ft_len: int, iters: int, prepopulate: int = 0, max_batch: int = 64,
        chunk: int = 512, max_tokens: int = 8192, max_ft_window: int = 8192,
        budget: Optional[float] = None, tpot_slo: float = 50.0, multi_layer: bool = False,
        policy: int = COSERVE, temporal_n: int = 128, rho: float = 0.5, gamma: float = 1.15):
    """coserve_loop.hpp run_coserve on the simulated clock.
    Returns the per-iteration log (list of dicts)."""
    budget = tpot_slo if budget is None else budget
    mem = MemoryModel(total_pages, page_size, growth)
    trace = generate_trace(w, seed)
    nxt = 0
    queue: deque = deque()
    running: List[Request] = []
    next_id = 0
    now = 0.0
    ft = FtState(L=ft_len, n_layers=n_layers)
    ft_pages = []
    if ft_len > 0:
        ft_pages = mem.reserve(mem.pages_for(ft_len))
        ft.phase, ft.minibatch = FWD, 0
    prng = TraceRng(seed ^ 0x5EED5EED)
    for _ in range(prepopulate):
        if len(running) >= max_batch:
            break
        p = clip_len(prng.lognormal(w.prompt_mu, w.prompt_sigma), w.prompt_min, w.prompt_max)
        g = clip_len(prng.lognormal(w.gen_mu, w.gen_sigma), w.gen_min, w.gen_max)
        r = Request(next_id, p, g, -1e18)
        next_id += 1
        r.prefilled = p
        r.emitted = 1 + prng.uniform_int(0, max(0, g - 2))
        r.first_token_ms = -1e18
        pages = mem.reserve(mem.pages_for(r.context() + 1 + growth))
        if pages is None:
            break
        r.pages = pages
        running.append(r)
    log = []
    temporal = policy in (TEMPORAL, DTS)
    spatial = policy in (SPATIAL, ISOLATE)           # baselines.hpp SpatialSplit
    g_int = 1.0 if policy == ISOLATE else gamma
    dts = DtsState()
    inf_since_ft, ft_block = 0, False
    for _ in range(iters):
        arrived = 0
        while nxt < len(trace) and trace[nxt][0] <= now:
            t, p, g = trace[nxt]
            nxt += 1
            queue.append(Request(next_id, p, g, t))
            next_id += 1
            arrived += 1
        i = 0
        while i < len(running):
            r = running[i]
            if not r.in_prefill() and not r.done() and r.context() + 1 > len(r.pages) * page_size:
                if not mem.grow(r.pages):
                    mem.release(r.pages)
                    r.pages = []
                    r.prefilled = 0
                    r.emitted = 0
                    queue.appendleft(r)
                    running.pop(i)
                    continue
            i += 1
        if spatial:
            idle = FtState(L=ft.L, n_layers=ft.n_layers, phase=0, minibatch=ft.minibatch,
                           l=ft.l, layer=ft.layer, lj=ft.lj)
            plan = plan_iteration(queue, running, idle, prof, max_batch, chunk, max_tokens,
                                  max_ft_window, mem, budget / (g_int / rho), multi_layer)
            tick = plan["pred"] * (g_int / rho) if plan["c"] > 0 else budget
            fplan = plan_iteration(deque(), [], ft, prof, max_batch, chunk, max_tokens,
                                   max_ft_window, mem, prof.t0_ms + tick * ((1.0 - rho) / g_int),
                                   multi_layer)
            for k in ("s", "phase", "layer", "l", "bwd"):
                plan[k] = fplan[k]
            plan["pred"] = tick
        elif not temporal:
            plan = plan_iteration(queue, running, ft, prof, max_batch, chunk, max_tokens,
                                  max_ft_window, mem, budget, multi_layer)
        elif ft_block:
            plan = plan_ft_block(ft, prof, max_tokens, max_ft_window)
        else:
            idle = FtState(L=ft.L, n_layers=ft.n_layers, phase=0, minibatch=ft.minibatch,
                           l=ft.l, layer=ft.layer, lj=ft.lj)
            plan = plan_iteration(queue, running, idle, prof, max_batch, chunk, max_tokens,
                                  max_ft_window, mem, budget, multi_layer)
            if plan["c"] == 0 and ft.L > 0:
                ft_block = True
                plan = plan_ft_block(ft, prof, max_tokens, max_ft_window)
        entry = {"c": plan["c"], "s": plan["s"], "phase": plan["phase"], "layer": plan["layer"],
                 "l": plan["l"], "n_decode": len(plan["decode"]), "n_prefill": len(plan["prefill"]),
                 "pred": plan["pred"], "bwd": plan["bwd"],
                 "decode_ids": [running[i].id for i in plan["decode"]],
                 "prefill": [(running[i].id, st, ln) for i, st, ln in plan["prefill"]],
                 "pages": {running[i].id: list(running[i].pages) for i in plan["decode"]}}
        now += plan["pred"]
        for i in plan["decode"]:
            r = running[i]
            r.emitted += 1
            if r.done():
                r.completion_ms = now
        for i, st, ln in plan["prefill"]:
            r = running[i]
            r.prefilled += ln
            if not r.in_prefill():
                r.emitted = 1
                r.first_token_ms = now
                if r.done():
                    r.completion_ms = now
        i = 0
        completed = 0
        while i < len(running):
            if running[i].done():
                mem.release(running[i].pages)
                running.pop(i)
                completed += 1
            else:
                i += 1
        if plan["phase"] == BWD:
            for (_, _, sw) in plan["bwd"]:
                advance_finetune(ft, sw)
        else:
            advance_finetune(ft, plan["s"])
        if temporal and not ft_block and ft.L > 0:
            inf_since_ft += 1
            if policy == TEMPORAL:
                ft_block = inf_since_ft >= max(1, temporal_n)
            else:
                ft_block = dts_step(dts, len(queue), len(plan["decode"]) + len(plan["prefill"]),
                                    arrived, completed)
        if ft.phase == DONE:
            ft_block, inf_since_ft = False, 0
            ft.phase, ft.minibatch, ft.l, ft.layer, ft.lj = FWD, ft.minibatch + 1, 0, 0, 0
        entry["t_ms"] = now
        entry["n_running"] = len(running)
        entry["n_queue"] = len(queue)
        log.append(entry)
    return log
