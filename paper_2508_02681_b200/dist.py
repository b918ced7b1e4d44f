"""One-process-per-GPU sharding of independent UNO-CG problems.

Config 3 (48 problems x 3 loads at 256^3) partitions into independent solves: no data-path
collective exists.  torch.distributed (NCCL on GPUs, gloo in CPU tests) is used only for
barriers, the max-over-ranks device time, sums of work counters and the final gather of the
small per-problem results (kappa_bar, iteration counts).
"""
from __future__ import annotations

import math
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


def eq27_cost(problem, tol: float = 1e-8, rho: float = 0.1) -> float:
    """Predicted PCG iterations of a config-3 problem (m, R) for the LPT shard: the Eq 27 bound
     2 C^m <= tol with C = (sqrt(cond) - 1)/(sqrt(cond) + 1) and the FANS condition
    bound cond <= R (1 + rho)/(1 - rho) of contrast R with the seeded perturbation rho (SURVEY
    §8(d) D2).  A scheduling heuristic only."""
    _, R = problem
    cond = max(R, 1.0 + 1e-12) * (1.0 + rho) / (1.0 - rho)
    C = (math.sqrt(cond) - 1.0) / (math.sqrt(cond) + 1.0)
    return math.log(tol / 2.0) / math.log(C)


def config3_problems(contrasts=(2.0, 5.0, 10.0, 20.0, 50.0, 100.0), n_micro: int = 8) -> list:
    """The fixed config-3 batch: 8 microstructures x 6 contrasts = 48 problems (m, R)."""
    return [(m, float(R)) for R in contrasts for m in range(n_micro)]


def config3_shard(world: int, rank: int, contrasts=(2.0, 5.0, 10.0, 20.0, 50.0, 100.0), n_micro: int = 8) -> list:
    """This rank's share of the fixed 48-problem config-3 batch: at 8 ranks the
    Latin square (rank g: microstructure (g + j) mod 8 with contrast j, j = 0..5 — every rank gets
    every contrast and 6 distinct microstructures); otherwise LPT on the Eq 27 cost; 1 rank: all."""
    probs = config3_problems(contrasts, n_micro)
    if world <= 1:
        return probs
    if world == n_micro and len(contrasts) <= n_micro:
        return [((rank + j) % n_micro, float(contrasts[j])) for j in range(len(contrasts))]
    return shard(probs, world, rank, cost=eq27_cost)


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
