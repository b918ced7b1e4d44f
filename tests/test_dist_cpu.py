"""Multi-process host logic of the batch sharding on CPU (gloo, world size 2): every problem is
owned by exactly one rank, LPT balances the Eq 27 cost, the max/sum reductions and the result
gather behave as bench.py relies on."""
import math
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2508_02681_b200 import dist as D
from paper_2508_02681_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _eq27_cost(p):
    # Eq 27 iteration bound with cond <= R * 1.1/0.9 for contrast R
    m, R = p
    cond = R * 1.1 / 0.9
    C = (math.sqrt(cond) - 1) / (math.sqrt(cond) + 1)
    return math.log(1e-8 / 2) / math.log(C)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    probs = [(m, R) for R in synth.CFG3_CONTRASTS for m in range(8)]
    mine = D.shard(probs, world, rank, cost=_eq27_cost)
    rr = D.shard(probs, world, rank)
    t = D.reduce_max(10.0 + rank)
    s = D.reduce_sum(len(mine))
    res = D.gather_results([{"p": p, "rank": rank} for p in mine])
    q.put((rank, mine, rr, t, s, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_sharding_and_reductions(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    probs = [(m, R) for R in synth.CFG3_CONTRASTS for m in range(8)]
    owned = sorted(p for _, mine, _, _, _, _ in outs for p in mine)
    assert owned == sorted(probs)                                   # partition, no overlap
    rr = sorted(p for _, _, rr, _, _, _ in outs for p in rr)
    assert rr == sorted(probs)
    loads = [sum(_eq27_cost(p) for p in mine) for _, mine, _, _, _, _ in outs]
    assert max(loads) / min(loads) < 1.02                          # LPT balance
    for rank, mine, _, t, s, res in outs:
        assert t == 10.0 + world - 1                                # max over ranks
        assert s == len(probs)                                      # sum over ranks
        assert [r["p"] for r in res] == [p for _, m, _, _, _, _ in outs for p in m]  # rank-ordered gather


def test_shard_single_rank_is_identity():
    probs = list(range(10))
    assert D.shard(probs, 1, 0) == probs
