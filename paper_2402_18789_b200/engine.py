"""Python mirror of the C ABI engine (include/coserve_cuda.h) for tests and bench.py.

`Engine` owns one cs_engine (one GPU).  Every method is a thin ctypes call into
libcoserve_cuda.so; errors follow the reference's conventions (ValueError for
std::invalid_argument, CacheDesync / OrderingViolation for SPEC.md:287,296).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib

i32, i64, f32, f64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_void_p

SEG_DECODE, SEG_PREFILL, SEG_FT_FWD = 0, 1, 2
FT_NONE, FT_FORWARD, FT_BACKWARD = 0, 1, 2


class ModelConfig(ctypes.Structure):
    _fields_ = [("n_layers", i32), ("hidden", i32), ("n_heads", i32), ("n_kv_heads", i32),
                ("head_dim", i32), ("ffn", i32), ("vocab", i32), ("lora_rank", i32),
                ("norm", i32), ("act", i32), ("rope", i32), ("qkv_bias", i32),
                ("rope_theta", f32), ("rms_eps", f32), ("page_size", i32), ("n_pages", i32),
                ("max_tokens", i32), ("max_ft_len", i32), ("max_segments", i32)]


class Segment(ctypes.Structure):
    _fields_ = [("kind", i32), ("q_start", i32), ("q_len", i32), ("ctx_start", i32),
                ("page_off", i32), ("n_pages", i32), ("sample", i32), ("adapter", i32)]


class FtWindow(ctypes.Structure):
    _fields_ = [("phase", i32), ("seq_len", i32), ("l", i32), ("s", i32), ("layer", i32),
                ("targets", ctypes.POINTER(i32)), ("page_off", i32), ("n_pages", i32)]


class IterationPlan(ctypes.Structure):
    _fields_ = [("n_tokens", i32), ("tokens", ctypes.POINTER(i32)), ("n_segments", i32),
                ("segments", ctypes.POINTER(Segment)), ("page_table", ctypes.POINTER(i32)),
                ("page_table_len", i32), ("ft", FtWindow), ("n_extra_bwd", i32),
                ("extra_bwd", ctypes.POINTER(FtWindow))]


class StepResult(ctypes.Structure):
    _fields_ = [("next_tokens", ctypes.POINTER(i32)), ("logits", ctypes.POINTER(f32)),
                ("ft_loss_sum", f64), ("iteration_ms", f32)]


class LatencyProfileC(ctypes.Structure):
    _fields_ = [("t0_ms", f64), ("slope_ms_per_token", f64), ("knee_tokens", f64),
                ("bwd_token_weight", f64), ("attn_fwd_ms_per_token_ctx", f64),
                ("attn_bwd_ms_per_token_ctx", f64), ("bwd_layer0_weight", f64),
                ("decode_ms_per_row", f64), ("prefill_ms_per_token", f64),
                ("fwd_window_ms", f64)]


class CoserveConfig(ctypes.Structure):
    _fields_ = [("rate_rps", f64), ("duration_s", f64), ("burst_amplitude", f64),
                ("burst_period_s", f64), ("tpot_slo_ms", f64), ("ttft_slo_ms", f64),
                ("budget_ms", f64), ("max_batch", i32), ("chunk_size", i32), ("max_tokens", i32),
                ("max_ft_window", i32), ("profile", LatencyProfileC), ("ft_seq_len", i32),
                ("growth_tokens", i32), ("warmup_iters", i32), ("timed_iters", i32),
                ("prepopulate", i32), ("adaptive", i32), ("profile_timed", i32),
                ("multi_layer_bwd", i32),
                ("seed", ctypes.c_uint64),
                ("n_layers", i32), ("vocab", i32), ("page_size", i32), ("total_pages", i64),
                ("policy", i32), ("temporal_n", i32), ("sim_clock", i32),
                ("vtc", i32), ("n_tenants", i32), ("ft_tenant", i32),
                ("tenant0_share", f64), ("vtc_wp", f64), ("vtc_wq", f64), ("vtc_wr", f64),
                ("tail_target", f64), ("spatial_rho", f64), ("spatial_gamma", f64)]

POLICY_COSERVE, POLICY_TEMPORAL, POLICY_DTS, POLICY_SPATIAL, POLICY_ISOLATE = 0, 1, 2, 3, 4


class CoserveStats(ctypes.Structure):
    _fields_ = [("iters", i64), ("timed_ms", f64), ("timed_device_ms", f64),
                ("ft_fwd_tokens", i64), ("ft_bwd_tokens", i64), ("ft_fwd_ms", f64),
                ("ft_bwd_ms", f64), ("minibatches_done", i64), ("inf_tokens", i64),
                ("gen_tokens", i64), ("requests_done", i64), ("requests_slo_ok", i64),
                ("evictions", i64), ("ttft_p50_ms", f64), ("ttft_p99_ms", f64),
                ("tpot_p50_ms", f64), ("tpot_p99_ms", f64), ("iter_p50_ms", f64),
                ("iter_p99_ms", f64), ("iter_max_ms", f64), ("gpu_launches", i64),
                ("h2d_bytes", i64), ("d2h_bytes", i64),
                ("tenant_service", f64 * 8), ("tenant_done", i64 * 8),
                ("vtc_spread_max", f64), ("vtc_pair_gap_max", f64),
                ("itl_p50_ms", f64), ("itl_p99_ms", f64), ("itl_max_ms", f64), ("itl_samples", i64),
                ("timed_arrivals", i64), ("timed_done", i64), ("timed_slo_ok", i64),
                ("timed_unfinished_miss", i64)]


class IterLogC(ctypes.Structure):
    _fields_ = [("t_ms", f64), ("pred_ms", f64), ("ms", f64), ("device_ms", f64), ("c", i32),
                ("s", i32), ("phase", i32), ("layer", i32), ("l", i32), ("n_decode", i32),
                ("n_prefill", i32), ("n_running", i32), ("n_queue", i32), ("timed", i32)]


def _declare_engine(L):
    P = ctypes.POINTER
    L.cs_engine_create.argtypes = [P(ModelConfig), ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                   P(vp)]
    L.cs_engine_destroy.argtypes = [vp]
    L.cs_engine_set_weight.argtypes = [vp, ctypes.c_char_p, ctypes.c_int, vp, ctypes.c_int, i64, i64]
    L.cs_engine_get_lora.argtypes = [vp, ctypes.c_int, vp, vp]
    L.cs_engine_init_random.argtypes = [vp, ctypes.c_uint64]
    L.cs_step.argtypes = [vp, P(IterationPlan), P(StepResult)]
    L.cs_step_async.argtypes = [vp, P(IterationPlan)]
    L.cs_sync.argtypes = [vp, P(StepResult)]
    L.cs_adam_step.argtypes = [vp, f32, f32, f32, f32]
    L.cs_zero_lora_grads.argtypes = [vp]
    L.cs_engine_reset_ft.argtypes = [vp]
    L.cs_engine_reset_ft.restype = ctypes.c_int
    L.cs_read_lora_grads.argtypes = [vp, ctypes.c_int, vp, vp]
    L.cs_read_kvgrad.argtypes = [vp, i32, vp, vp]
    L.cs_read_kv.argtypes = [vp, ctypes.c_int, vp, i32, vp, vp]
    L.cs_read_dy.argtypes = [vp, i32, vp]
    L.cs_coserve_run.restype = ctypes.c_int
    L.cs_coserve_run.argtypes = [vp, P(CoserveConfig), P(CoserveStats), P(IterLogC), i64, P(i64)]
    L.cs_engine_launch_count.restype = i64
    L.cs_engine_launch_count.argtypes = [vp]
    L.cs_engine_set_profiling.restype = ctypes.c_int
    L.cs_engine_set_profiling.argtypes = [vp, ctypes.c_int]
    L.cs_engine_read_profile.restype = ctypes.c_int
    L.cs_engine_read_profile.argtypes = [vp, ctypes.c_int, P(f64), P(f64), P(f64), P(i64)]
    L.cs_nccl_unique_id.argtypes = [vp]
    L.cs_tp_group_create.argtypes = [ctypes.c_int, P(vp)]
    L.cs_tp_group_destroy.argtypes = [vp]
    L.cs_engine_create_tp_local.argtypes = [P(ModelConfig), ctypes.c_int, ctypes.c_int, vp, P(vp)]
    L.cs_engine_create_ipc.argtypes = [P(ModelConfig), ctypes.c_int, ctypes.c_int, ctypes.c_int, P(vp)]
    L.cs_engine_ipc_handle.argtypes = [vp, vp, P(i64)]
    L.cs_engine_ipc_attach.argtypes = [vp, vp, vp]
    for name in ("cs_nccl_unique_id", "cs_tp_group_create", "cs_tp_group_destroy",
                 "cs_engine_create_tp_local", "cs_engine_create_ipc", "cs_engine_ipc_handle",
                 "cs_engine_ipc_attach"):
        getattr(L, name).restype = ctypes.c_int
    L.cs_engine_alloc_audit.restype = ctypes.c_int
    L.cs_engine_alloc_audit.argtypes = [vp, vp, vp, P(i64)]
    L.cs_engine_pool_info.restype = ctypes.c_int
    L.cs_engine_tp_sync_max.restype = ctypes.c_int
    L.cs_engine_tp_sync_max.argtypes = [vp, P(f64), ctypes.c_int]
    L.cs_engine_pool_info.argtypes = [vp, P(i32), P(i32), P(i32), P(i64)]
    L.cs_sched_latency.restype = f64
    L.cs_sched_latency.argtypes = [P(LatencyProfileC), i64, i64]
    L.cs_sched_max_finetune_tokens.restype = i64
    L.cs_sched_max_finetune_tokens.argtypes = [P(LatencyProfileC), i64, f64]
    for name in ("cs_engine_create", "cs_engine_destroy", "cs_engine_set_weight",
                 "cs_engine_get_lora", "cs_engine_init_random", "cs_step", "cs_step_async",
                 "cs_sync", "cs_adam_step", "cs_zero_lora_grads", "cs_read_lora_grads",
                 "cs_read_kvgrad", "cs_read_kv", "cs_read_dy"):
        getattr(L, name).restype = ctypes.c_int


_DECLARED = False


def lib():
    global _DECLARED
    L = _lib.lib()
    if not _DECLARED:
        _declare_engine(L)
        _DECLARED = True
    return L


@dataclass
class Seg:
    """One segment of the mixed token batch (cs_segment)."""
    kind: int
    tokens: Sequence[int]
    ctx_start: int
    pages: Sequence[int]
    sample: bool = False
    adapter: bool = False


def arch_config(arch, page_size=16, n_pages=256, max_tokens=256, max_ft_len=256,
                max_segments=64) -> ModelConfig:
    """ModelConfig from an oracle.Arch-like object (fields n_layers, hidden, ...)."""
    c = ModelConfig()
    c.n_layers = arch.n_layers
    c.hidden = arch.hidden
    c.n_heads = arch.n_heads
    c.n_kv_heads = arch.n_kv_heads
    c.head_dim = arch.head_dim
    c.ffn = arch.ffn
    c.vocab = arch.vocab
    c.lora_rank = arch.lora_rank
    c.norm = 1 if arch.norm == "rms" else 0
    c.act = 1 if arch.act == "swiglu" else 0
    c.rope = 1 if arch.rope else 0
    c.qkv_bias = 1 if arch.qkv_bias else 0
    c.rope_theta = arch.rope_theta
    c.rms_eps = arch.rms_eps
    c.page_size = page_size
    c.n_pages = n_pages
    c.max_tokens = max_tokens
    c.max_ft_len = max_ft_len
    c.max_segments = max_segments
    return c


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it; the host shares it, e.g. by torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    _lib.check(lib().cs_nccl_unique_id(buf), "cs_nccl_unique_id")
    return buf.raw


class TPGroup:
    """Single-process tensor-parallel group (cs_tp_group): engines of this process, one host
    thread each, all-reduce by the one-shot peer kernel.  Destroy after its engines."""

    def __init__(self, size: int):
        self._L = lib()
        h = vp()
        _lib.check(self._L.cs_tp_group_create(size, ctypes.byref(h)), "cs_tp_group_create")
        self._h = h
        self.size = size

    def close(self):
        if getattr(self, "_h", None):
            self._L.cs_tp_group_destroy(self._h)
            self._h = None


def tp_run(engines: Sequence["Engine"], fn):
    """Run fn(engine) on every rank concurrently (one thread per rank, as cs_step requires
    for a TP group); returns the per-rank results, re-raising the first failure."""
    import threading
    out = [None] * len(engines)
    err = [None] * len(engines)

    def body(i):
        try:
            out[i] = fn(engines[i])
        except BaseException as ex:  # noqa: BLE001 -- re-raised below
            err[i] = ex
    th = [threading.Thread(target=body, args=(i,)) for i in range(len(engines))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


class Engine:
    def __init__(self, cfg: ModelConfig, device: int = 0, tp_rank: int = 0, tp_size: int = 1,
                 group: Optional[TPGroup] = None, nccl_uid: Optional[bytes] = None,
                 ipc: bool = False):
        """tp_size > 1: group -> single-process peer group; ipc -> cross-process CUDA-IPC peer
        group (attach with tp_ipc.connect); else NCCL from nccl_uid."""
        self.cfg = cfg
        self._L = lib()
        self.tp_rank = tp_rank
        self.tp_size = group.size if group is not None else tp_size
        h = vp()
        if group is not None:
            _lib.check(self._L.cs_engine_create_tp_local(ctypes.byref(cfg), device, tp_rank,
                                                         group._h, ctypes.byref(h)),
                       "cs_engine_create_tp_local")
        elif ipc:
            _lib.check(self._L.cs_engine_create_ipc(ctypes.byref(cfg), device, tp_rank, tp_size,
                                                    ctypes.byref(h)), "cs_engine_create_ipc")
        else:
            uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid else None
            _lib.check(self._L.cs_engine_create(ctypes.byref(cfg), device, tp_rank, tp_size, uid,
                                                ctypes.byref(h)), "cs_engine_create")
        self._h = h
        # this rank's shard sizes
        self.ffn_local = cfg.ffn // self.tp_size
        self.kv_dim_local = cfg.n_kv_heads // self.tp_size * cfg.head_dim

    def close(self):
        if getattr(self, "_h", None):
            self._L.cs_engine_destroy(self._h)
            self._h = None

    # -------------------------------------------------------------- IPC peer group
    def ipc_handle(self):
        """(64-byte CUDA IPC handle of this rank's engine arena, arena bytes)."""
        buf = ctypes.create_string_buffer(64)
        n = i64()
        _lib.check(self._L.cs_engine_ipc_handle(self._h, buf, ctypes.byref(n)), "cs_engine_ipc_handle")
        return buf.raw, n.value

    def ipc_attach(self, handles: Sequence[bytes], arena_bytes: Sequence[int]):
        """Map the other ranks' arenas (handles / sizes in tp-rank order)."""
        if len(handles) != self.tp_size or any(len(h) != 64 for h in handles):
            raise ValueError("ipc_attach: one 64-byte handle per tp rank")
        hb = ctypes.create_string_buffer(b"".join(handles), 64 * self.tp_size)
        sz = (i64 * self.tp_size)(*arena_bytes)
        _lib.check(self._L.cs_engine_ipc_attach(self._h, hb, sz), "cs_engine_ipc_attach")

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- weights
    def set_weight(self, name: str, layer: int, value: np.ndarray):
        v = np.ascontiguousarray(value, dtype=np.float64)
        if v.ndim == 1:
            v = v.reshape(1, -1)
        _lib.check(self._L.cs_engine_set_weight(self._h, name.encode(), layer, v.ctypes.data, 0,
                                                v.shape[0], v.shape[1]), f"set_weight({name})")

    def load_weights(self, W: Dict):
        """W in the oracle's dict format (reference layouts)."""
        self.set_weight("embed", 0, W["embed"])
        self.set_weight("unembed", 0, W["unembed"])
        if "gf" in W:
            self.set_weight("final_norm", 0, W["gf"])
        names = {"wq": "wq", "wk": "wk", "wv": "wv", "wo": "wo", "w_gate": "w_gate",
                 "w_up": "w_up", "w_down": "w_down", "lora_a": "lora_a", "lora_b": "lora_b",
                 "bq": "bq", "bk": "bk", "bv": "bv", "g1": "norm1", "g2": "norm2"}
        for l, Lw in enumerate(W["layers"]):
            for k, v in Lw.items():
                self.set_weight(names[k], l, v)

    def init_random(self, seed: int = 1):
        _lib.check(self._L.cs_engine_init_random(self._h, seed), "init_random")

    # -------------------------------------------------------------- step
    def _plan(self, segs: List[Seg], ft: Optional[Dict]):
        tokens, cs_segs, pt = [], [], []
        row = 0
        for s in segs:
            g = Segment()
            g.kind = s.kind
            g.q_start = row
            g.q_len = len(s.tokens)
            g.ctx_start = s.ctx_start
            g.page_off = len(pt)
            g.n_pages = len(s.pages)
            g.sample = 1 if s.sample else 0
            g.adapter = 1 if s.adapter else 0
            pt.extend(int(p) for p in s.pages)
            tokens.extend(int(t) for t in s.tokens)
            cs_segs.append(g)
            row += g.q_len
        w = FtWindow()
        keep = {}
        if ft:
            w.phase = ft["phase"]
            w.seq_len = ft.get("seq_len", 0)
            w.l = ft.get("l", 0)
            w.s = ft.get("s", 0)
            w.layer = ft.get("layer", 0)
            if "pages" in ft:
                w.page_off = len(pt)
                w.n_pages = len(ft["pages"])
                pt.extend(int(p) for p in ft["pages"])
            if "targets" in ft:
                tg = np.ascontiguousarray(ft["targets"], dtype=np.int32)
                keep["tg"] = tg
                w.targets = tg.ctypes.data_as(ctypes.POINTER(i32))
        extra = []
        if ft and ft.get("extra"):
            for x in ft["extra"]:
                e = FtWindow()
                e.phase, e.seq_len, e.l, e.s, e.layer = FT_BACKWARD, w.seq_len, x["l"], x["s"], x["layer"]
                e.page_off, e.n_pages = w.page_off, w.n_pages
                extra.append(e)
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        ptab = np.ascontiguousarray(pt if pt else [0], dtype=np.int32)
        seg_arr = (Segment * max(1, len(cs_segs)))(*cs_segs)
        p = IterationPlan()
        p.n_tokens = len(tokens)
        p.tokens = tok.ctypes.data_as(ctypes.POINTER(i32))
        p.n_segments = len(cs_segs)
        p.segments = seg_arr
        p.page_table = ptab.ctypes.data_as(ctypes.POINTER(i32))
        p.page_table_len = len(pt)
        p.ft = w
        if extra:
            ex_arr = (FtWindow * len(extra))(*extra)
            p.n_extra_bwd = len(extra)
            p.extra_bwd = ex_arr
            keep["extra"] = ex_arr
        keep.update(tok=tok, ptab=ptab, segs=seg_arr)
        return p, keep

    def step(self, segs: List[Seg], ft: Optional[Dict] = None, want_logits: bool = False):
        p, keep = self._plan(segs, ft)
        n_s = sum(1 for s in segs if s.sample)
        nt = np.full(max(1, len(segs)), -1, dtype=np.int32)
        logits = np.zeros((max(1, n_s), self.cfg.vocab), dtype=np.float32) if want_logits else None
        r = StepResult()
        r.next_tokens = nt.ctypes.data_as(ctypes.POINTER(i32))
        if logits is not None:
            r.logits = logits.ctypes.data_as(ctypes.POINTER(f32))
        _lib.check(self._L.cs_step(self._h, ctypes.byref(p), ctypes.byref(r)), "cs_step")
        del keep
        out = {"next_tokens": nt[:len(segs)], "loss_sum": r.ft_loss_sum, "ms": r.iteration_ms}
        if logits is not None:
            out["logits"] = logits[:n_s]
        return out

    def step_async(self, segs: List[Seg], ft: Optional[Dict] = None):
        p, keep = self._plan(segs, ft)
        _lib.check(self._L.cs_step_async(self._h, ctypes.byref(p)), "cs_step_async")
        return keep

    def sync(self) -> float:
        r = StepResult()
        _lib.check(self._L.cs_sync(self._h, ctypes.byref(r)), "cs_sync")
        return r.iteration_ms

    def adam_step(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        _lib.check(self._L.cs_adam_step(self._h, lr, beta1, beta2, eps), "cs_adam_step")

    def reset_ft(self):
        _lib.check(self._L.cs_engine_reset_ft(self._h), "reset_ft")

    def zero_lora_grads(self):
        _lib.check(self._L.cs_zero_lora_grads(self._h), "zero_lora_grads")

    # -------------------------------------------------------------- read-back
    def lora_grads(self, layer: int):
        """(dA, dB) of this rank: dA rows = its ffn shard; dB = its partial sum (TP)."""
        c = self.cfg
        a = np.zeros((self.ffn_local, c.lora_rank))
        b = np.zeros((c.lora_rank, c.hidden))
        _lib.check(self._L.cs_read_lora_grads(self._h, layer, a.ctypes.data, b.ctypes.data), "read_lora_grads")
        return a, b

    def lora(self, layer: int):
        c = self.cfg
        a = np.zeros((self.ffn_local, c.lora_rank))
        b = np.zeros((c.lora_rank, c.hidden))
        _lib.check(self._L.cs_engine_get_lora(self._h, layer, a.ctypes.data, b.ctypes.data), "get_lora")
        return a, b

    def kvgrad(self, L: int):
        kv = self.kv_dim_local
        dk = np.zeros((L, kv))
        dv = np.zeros((L, kv))
        _lib.check(self._L.cs_read_kvgrad(self._h, L, dk.ctypes.data, dv.ctypes.data), "read_kvgrad")
        return dk, dv

    def read_kv(self, layer: int, pages: Sequence[int], length: int):
        kv = self.kv_dim_local
        pg = np.ascontiguousarray(pages, dtype=np.int32)
        k = np.zeros((length, kv))
        v = np.zeros((length, kv))
        _lib.check(self._L.cs_read_kv(self._h, layer, pg.ctypes.data, length, k.ctypes.data,
                                      v.ctypes.data), "read_kv")
        return k, v

    def set_profiling(self, on: bool):
        _lib.check(self._L.cs_engine_set_profiling(self._h, 1 if on else 0), "set_profiling")

    def read_profile(self, kind: int) -> Dict:
        ms, fl, by, n = f64(), f64(), f64(), i64()
        _lib.check(self._L.cs_engine_read_profile(self._h, kind, ctypes.byref(ms), ctypes.byref(fl),
                                                  ctypes.byref(by), ctypes.byref(n)), "read_profile")
        return {"ms": ms.value, "flops": fl.value, "bytes": by.value, "launches": n.value}

    def alloc_audit(self):
        """[(name, elements, elem_bytes)] of every device buffer + transient allocation count
        (cs_engine_alloc_audit, the Matrix::alloc_hook analogue)."""
        recs = []
        HOOK = ctypes.CFUNCTYPE(None, ctypes.c_char_p, i64, i32, vp)
        cb = HOOK(lambda n, el, b, u: recs.append((n.decode(), int(el), int(b))))
        tr = i64()
        _lib.check(self._L.cs_engine_alloc_audit(self._h, ctypes.cast(cb, vp), None, ctypes.byref(tr)),
                   "alloc_audit")
        return recs, tr.value

    def tp_sync_max(self, vals: Sequence[float]) -> List[float]:
        """Max over this engine's TP group (every rank calls it; identity at tp_size 1)."""
        buf = (f64 * len(vals))(*vals)
        _lib.check(self._L.cs_engine_tp_sync_max(self._h, buf, len(vals)), "tp_sync_max")
        return list(buf)

    def launch_count(self) -> int:
        return int(self._L.cs_engine_launch_count(self._h))

    def read_dy(self, L: int):
        out = np.zeros((L, self.cfg.hidden))
        _lib.check(self._L.cs_read_dy(self._h, L, out.ctypes.data), "read_dy")
        return out


def _struct_dict(st) -> Dict:
    out = {}
    for name, _ in st._fields_:
        v = getattr(st, name)
        out[name] = list(v) if isinstance(v, ctypes.Array) else v
    return out


def coserve_run(engine: Optional["Engine"], cfg: CoserveConfig, log_cap: int = 100000):
    """cs_coserve_run: the C++ co-serving loop (engine=None -> simulated clock)."""
    L = lib()
    stats = CoserveStats()
    log = (IterLogC * max(1, log_cap))()
    n = i64(0)
    rc = L.cs_coserve_run(engine._h if engine is not None else None, ctypes.byref(cfg),
                          ctypes.byref(stats), log, log_cap, ctypes.byref(n))
    _lib.check(rc, "cs_coserve_run")
    return _struct_dict(stats), [_struct_dict(log[i]) for i in range(n.value)]


def profile_struct(t0_ms, slope, knee=0.0, bwd_weight=1.0, attn_fwd=0.0, attn_bwd=0.0,
                   layer0_weight=1.0, decode_row=0.0, prefill_token=0.0,
                   fwd_window=0.0) -> LatencyProfileC:
    p = LatencyProfileC()
    p.fwd_window_ms = fwd_window
    p.t0_ms, p.slope_ms_per_token, p.knee_tokens, p.bwd_token_weight = t0_ms, slope, knee, bwd_weight
    p.attn_fwd_ms_per_token_ctx, p.attn_bwd_ms_per_token_ctx = attn_fwd, attn_bwd
    p.bwd_layer0_weight = layer0_weight
    p.decode_ms_per_row, p.prefill_ms_per_token = decode_row, prefill_token
    return p


def sched_latency(t0_ms, slope, knee, c, s) -> float:
    p = profile_struct(t0_ms, slope, knee)
    return lib().cs_sched_latency(ctypes.byref(p), c, s)


def sched_max_finetune_tokens(t0_ms, slope, knee, c, slo_ms) -> int:
    p = profile_struct(t0_ms, slope, knee)
    return lib().cs_sched_max_finetune_tokens(ctypes.byref(p), c, slo_ms)
