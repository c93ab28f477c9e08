"""Cross-process peer-memory tensor parallelism (cs_engine_create_ipc + tp_ipc.connect): one
process per rank, the ranks' engine arenas mapped with CUDA IPC handles exchanged through
torch.distributed, the fused row-parallel GEMM + all-reduce and the one-shot all-reduces over
peer memory, ordered by the device-side flag barrier -- bench.py --tp T under torchrun
(parallelize.hpp:50-53 cost form; SURVEY.md §8e layout).

CPU (gloo, world size 4 = two TP groups of 2): the handle exchange itself -- every rank gets
its own group's handles in tp-rank order, a missing rank is an error.
GPU (one B200): two processes on the same device form one TP=2 group; their results against
the oracle (same gates as tests/test_tp.py) and against each other (replicated head and B
bit-identical)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import coserve_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _FakeEngine:
    def __init__(self, tp_rank, tp_size, tag):
        self.tp_rank, self.tp_size, self.tag = tp_rank, tp_size, tag
        self.attached = None

    def ipc_handle(self):
        return bytes([self.tag]) * 64, 1 << 30

    def ipc_attach(self, handles, sizes):
        self.attached = (handles, sizes)


def _exchange_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_18789_b200 import tp_ipc
    tp = 2
    group, tp_rank = rank // tp, rank % tp
    e = _FakeEngine(tp_rank, tp, tag=16 * group + tp_rank)
    tp_ipc.connect(e, dist, group)
    bad = None
    try:  # a group whose ranks do not cover 0..tp-1 must not attach
        tp_ipc.gather_group_handles(dist, group, 0, tp, b"x" * 64, 1)
    except RuntimeError as ex:
        bad = str(ex)
    q.put((rank, [h[0] for h in e.attached[0]], e.attached[1], bad))
    dist.destroy_process_group()


def test_ipc_handle_exchange_gloo():
    world, port = 4, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tags, sizes, bad in res:
        g = rank // 2
        assert tags == [16 * g, 16 * g + 1]          # own group, tp-rank order
        assert sizes == [1 << 30, 1 << 30]
        assert bad is not None and "ranks" in bad    # rank 0 claimed twice -> rejected


# ------------------------------------------------------------------------------------- GPU
def _gpu_worker(rank, port, q, fused):
    os.environ["CS_TP_FUSED"] = fused
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2402_18789_b200 import tp_ipc
    from paper_2402_18789_b200.engine import Engine, arch_config
    from tests.test_tp import ARCH, _plan_steps
    arch = ARCH
    W = O.init_general(arch, 3)
    toks = list(np.random.default_rng(5).integers(0, arch.vocab, 100))
    steps, _ = _plan_steps(arch, toks, [40, 60], [30, 30, 40], n_inf=5, seed=7, P=16)
    cfg = arch_config(arch, page_size=16, n_pages=256, max_tokens=512, max_ft_len=100,
                      max_segments=64)
    e = Engine(cfg, device=0, tp_rank=rank, tp_size=2, ipc=True)
    tp_ipc.connect(e, dist, 0)
    e.load_weights(W)
    out = {"logits": [], "next": [], "loss": 0.0, "kvg": {}}
    for kind, segs, ft, extra in steps:
        o = e.step(segs, ft=ft, want_logits=(kind != "bwd"))
        if kind == "bwd":
            if extra > 0 and ft["l"] - ft["s"] == 0:
                out["kvg"][extra] = e.kvgrad(len(toks))
            continue
        out["logits"].append(o["logits"])
        out["next"].append(o["next_tokens"])
        if kind == "fwd":
            out["loss"] += o["loss_sum"]
    out["grads"] = [e.lora_grads(l) for l in range(arch.n_layers)]
    e.adam_step(1e-3)
    out["B_after"] = [e.lora(l)[1] for l in range(arch.n_layers)]
    e.close()
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("fused", ["1", "0"])
def test_tp2_ipc_two_processes_match_oracle(fused):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, port, q, fused)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = dict(q.get(timeout=600) for _ in range(2))
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    from tests.test_tp import ARCH, _plan_steps
    arch = ARCH
    W = O.init_general(arch, 3)
    toks = list(np.random.default_rng(5).integers(0, arch.vocab, 100))
    tr = O.forward_full(arch, W, toks)
    bw = O.backward_full(arch, W, tr)
    steps, reqs = _plan_steps(arch, toks, [40, 60], [30, 30, 40], n_inf=5, seed=7, P=16)
    r0, r1 = res[0], res[1]
    for a, b in zip(r0["logits"], r1["logits"]):     # replicated head: bit-identical
        assert np.abs(a - b).max() == 0.0
    for a, b in zip(r0["next"], r1["next"]):
        np.testing.assert_array_equal(a, b)
    caches = [O.QkvCache(arch, r["len"] + 8) for r in reqs]
    diffs = []
    k = 0
    for kind, segs, ft, extra in steps:
        if kind == "bwd":
            continue
        for i, (tk, pos) in enumerate(extra):
            lg, _ = O.forward_window(arch, W, tk, pos, caches[i], lora=False)
            diffs.append(O.scaled_err(r0["logits"][k][i], lg[-1]))
        k += 1
    assert max(diffs) < 0.04, max(diffs)
    assert O.rel_err(r0["loss"] / 99.0, tr["loss"]) < 1e-2
    for l in range(arch.n_layers):
        ga = np.concatenate([r0["grads"][l][0], r1["grads"][l][0]], axis=0)
        gb = r0["grads"][l][1] + r1["grads"][l][1]   # folded LoRA: per-rank partial dB
        floor = 0.02 if l == arch.n_layers - 1 else 0.08
        assert O.scaled_err(ga, bw["grads"]["a"][l]) < floor, l
        assert O.scaled_err(gb, bw["grads"]["b"][l]) < floor, l
        assert np.abs(r0["B_after"][l] - r1["B_after"][l]).max() == 0.0   # dB all-reduced in Adam
    for n in (1, 2):
        dk = np.concatenate([r0["kvg"][n][0], r1["kvg"][n][0]], axis=1)
        dv = np.concatenate([r0["kvg"][n][1], r1["kvg"][n][1]], axis=1)
        assert O.scaled_err(dk, bw["layers"][n]["dk"]) < 0.08, n
        assert O.scaled_err(dv, bw["layers"][n]["dv"]) < 0.08, n
