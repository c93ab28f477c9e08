"""Multi-GPU aggregation for bench.py: one process per GPU, each an independent co-serving
replica (TP=1 pipelines for the 8B model).  There is no data-path
collective; only the timing reduction: value = sum of per-replica finetuning units / max
over ranks of the timed region (weak scaling).  With bench.py --tp T, T consecutive ranks form
one tensor-parallel replica (collectives inside the step) and count once."""
from __future__ import annotations

from typing import Dict, Tuple


def ft_rate_per_ms(st: Dict, n_layers: int) -> float:
    """Finetuning mini-batch progress in tokens/ms: L / t_mb with
    t_mb = L/r_f + N*L/r_b from the measured forward / backward window rates."""
    f, b = st["ft_fwd_tokens"], st["ft_bwd_tokens"]
    fm, bm = st["ft_fwd_ms"], st["ft_bwd_ms"]
    if f > 0 and b > 0 and fm > 0 and bm > 0:
        return 1.0 / (1.0 / (f / fm) + n_layers / (b / bm))
    tot = st["timed_device_ms"]
    return ((f + b / n_layers) / 2.0) / tot if tot > 0 else 0.0


def aggregate(st: Dict, n_layers: int, dist=None, device="cpu",
              count: bool = True) -> Tuple[float, float]:
    """Returns (value, e2e) in tokens/s over all ranks: units summed, time = max over ranks.
    count=False: this rank's units are not added (a non-leader rank of a tensor-parallel
    group, whose finetuning progress is its leader's)."""
    import torch
    rate_dev = ft_rate_per_ms(st, n_layers) if count else 0.0
    wall_factor = st["timed_device_ms"] / st["timed_ms"] if st["timed_ms"] > 0 else 1.0
    t = torch.tensor([st["timed_device_ms"], st["timed_ms"]], dtype=torch.float64, device=device)
    u = torch.tensor([rate_dev * st["timed_device_ms"], rate_dev * wall_factor * st["timed_ms"]],
                     dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
    dev_ms, wall_ms = t.tolist()
    units_dev, units_wall = u.tolist()
    value = 1000.0 * units_dev / dev_ms if dev_ms > 0 else 0.0
    e2e = 1000.0 * units_wall / wall_ms if wall_ms > 0 else 0.0
    return value, e2e
