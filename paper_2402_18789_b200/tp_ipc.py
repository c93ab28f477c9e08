"""Host side of the cross-process peer-memory TP group (cs_engine_create_ipc): the ranks'
CUDA IPC handles travel through torch.distributed (any backend -- gloo on CPU is enough) and
every engine maps its group's peer arenas.  The ranks of one TP group are `tp` consecutive
global ranks (bench.py --tp); several groups may share one process group."""
from __future__ import annotations

from typing import List, Sequence, Tuple


def gather_group_handles(dist, group_id: int, tp_rank: int, tp: int, handle: bytes,
                         arena_bytes: int) -> Tuple[List[bytes], List[int]]:
    """All-gather (group, tp rank, handle, bytes) over the world; return this group's handles
    and arena sizes in tp-rank order.  Raises if a rank of the group is missing or doubled."""
    world = dist.get_world_size()
    rec = [None] * world
    dist.all_gather_object(rec, (int(group_id), int(tp_rank), bytes(handle), int(arena_bytes)))
    mine = sorted((r for r in rec if r[0] == group_id), key=lambda r: r[1])
    if [r[1] for r in mine] != list(range(tp)):
        raise RuntimeError(f"tp group {group_id}: ranks {[r[1] for r in mine]} != 0..{tp - 1}")
    return [r[2] for r in mine], [r[3] for r in mine]


def connect(engine, dist, group_id: int = 0) -> None:
    """Exchange the group's IPC handles and attach `engine` (every rank of the world calls it
    collectively, after creating its engine with ipc=True)."""
    h, n = engine.ipc_handle()
    handles, sizes = gather_group_handles(dist, group_id, engine.tp_rank, engine.tp_size, h, n)
    engine.ipc_attach(handles, sizes)
