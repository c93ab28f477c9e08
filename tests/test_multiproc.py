"""N>1 path of bench.py on CPU: world_size-2 gloo, each rank an independent replica running
the C++ co-serving loop on the simulated clock; the timing reduction must equal the sum of
replica units over the max-over-ranks time."""
import os
import socket

import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import scheduler_oracle as S
    from paper_2402_18789_b200 import engine as E
    from paper_2402_18789_b200.replicas import aggregate, ft_rate_per_ms
    from tests.test_scheduler import _cfg
    prof = S.Profile(5.0, 0.01, S.INF, 0.05)
    st, _ = E.coserve_run(None, _cfg(20.0, prof, 300, 1024, 8, seed=rank))
    val, e2e = aggregate(st, 8, dist)
    q.put((rank, st["timed_device_ms"], ft_rate_per_ms(st, 8), val, e2e))
    dist.destroy_process_group()


def test_two_replicas_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tmax = max(r[1] for r in res)
    expect = 1000.0 * sum(r[2] * r[1] for r in res) / tmax
    for r in res:
        assert abs(r[3] - expect) < 1e-6 * expect      # every rank agrees on the value
    assert res[0][3] > 0.9 * 1000.0 * (res[0][2] + res[1][2])  # ~linear in replicas


def _tp_worker(rank, world, port, q):
    """Both ranks form ONE tensor-parallel replica (bench.py --tp 2): rank-identical loops
    (the simulated clock stands in for the max-reduced GPU clock) and only the leader counts."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import scheduler_oracle as S
    from paper_2402_18789_b200 import engine as E
    from paper_2402_18789_b200.replicas import aggregate, ft_rate_per_ms
    from tests.test_scheduler import _cfg
    prof = S.Profile(5.0, 0.01, S.INF, 0.05)
    st, log = E.coserve_run(None, _cfg(20.0, prof, 300, 1024, 8, seed=0))
    val, e2e = aggregate(st, 8, dist, count=(rank == 0))
    q.put((rank, ft_rate_per_ms(st, 8), val, [(g["c"], g["s"], g["layer"]) for g in log]))
    dist.destroy_process_group()


def test_tp_group_counts_once_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][3] == res[1][3]                   # the ranks planned identical iterations
    for r in res:
        assert abs(r[2] - 1000.0 * res[0][1]) < 1e-6 * r[2]   # one replica's rate, not two
