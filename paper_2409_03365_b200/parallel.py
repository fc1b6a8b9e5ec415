"""Sharding of independent planning problems across ranks and the global
best-plan exchange.

* Problems (sweep mixtures, candidate plans) are independent.  A fixed set is
  split strided: rank r of P plans global indices i with i % P == r (per-plan
  cost changes with the device count every 45 sweep indices).  Weak scaling
  gives every rank its own contiguous block of `per_rank` indices (the sweep
  pattern repeats every 180 indices, so every block has the same mix).  No
  collective on the data path.
* One exchange at the end: the global best plan = argmin over (key, global
  index); infeasible plans carry +inf.  NCCL has no MINLOC, so each rank
  contributes a 16-byte {key, index} record to one all_gather over NVLink and
  every rank reduces the P records locally (ties -> smaller index).
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist


def shard(total: int, rank: int, world: int) -> range:
    """Global problem indices owned by `rank` (strided assignment)."""
    return range(rank, total, world)


def local_to_global(local_index: int, rank: int, world: int) -> int:
    return rank + local_index * world


def block(per_rank: int, rank: int) -> range:
    """Global problem indices owned by `rank` under weak scaling (one block per rank)."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def block_to_global(local_index: int, rank: int, per_rank: int) -> int:
    return rank * per_rank + local_index


def reduce_minloc(records: list[tuple[float, int]]) -> tuple[float, int]:
    """argmin over (key, index); NaN/+inf keys lose; ties -> smaller index."""
    best_k, best_i = math.inf, -1
    for k, i in records:
        if i < 0 or not (k == k):
            continue
        if best_i < 0 or k < best_k or (k == best_k and i < best_i):
            best_k, best_i = k, i
    return best_k, best_i


def global_best(local_key: float, local_global_index: int, device: torch.device | None = None) -> tuple[float, int]:
    """All-gather every rank's local best {key, global index} and min-loc them.

    With the NCCL backend the 16-byte records travel over NVLink/NVSwitch; with
    gloo (CPU tests) over TCP.  Returns the same (key, index) on every rank.
    """
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return reduce_minloc([(local_key, local_global_index)])
    rec = torch.tensor([local_key, float(local_global_index)], dtype=torch.float64,
                       device=device if device is not None else "cpu")
    out = [torch.empty_like(rec) for _ in range(dist.get_world_size())]
    dist.all_gather(out, rec)
    return reduce_minloc([(float(t[0]), int(t[1])) for t in out])
