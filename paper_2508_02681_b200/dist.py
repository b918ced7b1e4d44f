"""One-process-per-GPU sharding of independent UNO-CG problems.

Config 3 (48 problems x 3 loads at 256^3) partitions into independent solves: no data-path
collective exists.  torch.distributed (NCCL on GPUs, gloo in CPU tests) is used only for
barriers, the max-over-ranks device time, sums of work counters and the final gather of the
small per-problem results (kappa_bar, iteration counts).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(problems: list, world: int, rank: int, cost=None) -> list:
    """Problems owned by `rank`.  With a cost predictor (e.g. the Eq 27 iteration bound) the
    assignment is LPT (largest cost first onto the least-loaded rank, ties by rank); without
    one it is round-robin.  Deterministic on every rank."""
    if world <= 1:
        return list(problems)
    if cost is None:
        return [p for i, p in enumerate(problems) if i % world == rank]
    order = sorted(range(len(problems)), key=lambda i: (-cost(problems[i]), i))
    load = [0.0] * world
    owner = {}
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[i] = r
        load[r] += cost(problems[i])
    return [problems[i] for i in range(len(problems)) if owner[i] == rank]


def _device_for_backend():
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def reduce_max(x: float) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_results(local: list) -> list:
    """All ranks' small result records (picklable), concatenated in rank order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(local)
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, list(local))
    return [x for part in out for x in part]
