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
    mine = D.config3_shard(world, rank)  # bench.py's assignment of the fixed 48-problem batch
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


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_config3_shard_partitions_the_fixed_batch(world):
    # every (microstructure, contrast) pair of the 48-problem batch is solved by exactly one rank;
    # 8 ranks: Latin square (every rank all six contrasts, six distinct microstructures);
    # 2/4 ranks: LPT on the Eq 27 cost, balanced to 2 %
    probs = [(m, R) for R in synth.CFG3_CONTRASTS for m in range(8)]
    parts = [D.config3_shard(world, r) for r in range(world)]
    assert sorted(p for part in parts for p in part) == sorted(probs)
    assert D.config3_problems() == probs
    if world == 8:
        for part in parts:
            assert sorted(R for _, R in part) == sorted(synth.CFG3_CONTRASTS)
            assert len({m for m, _ in part}) == 6
            assert [(m, j) for (m, _), j in zip(part, range(6))] == \
                [a for a in synth.config3_assignment(8, parts.index(part))]
    cost = [sum(D.eq27_cost(p) for p in part) for part in parts]
    assert max(cost) / min(cost) < 1.02
    assert abs(D.eq27_cost((0, 100.0)) - _eq27_cost((0, 100.0))) < 1e-9


def test_shard_single_rank_is_identity():
    probs = list(range(10))
    assert D.shard(probs, 1, 0) == probs


# ----------------------------------------------------------------------------- slab exchanges
def _slab_bufs(rank, world, blk=6, hs=5):
    import torch

    g = torch.Generator().manual_seed(100 + rank)
    send = torch.randn((world, blk), generator=g, dtype=torch.float64)
    hsend = torch.randn((2, hs), generator=g, dtype=torch.float64)
    red = torch.randn(3, generator=g, dtype=torch.float64)
    return send, hsend, red


def _slab_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2508_02681_b200.slab import MAX, SUM, DistComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = DistComm()
    send, hsend, red = _slab_bufs(rank, world)
    recv = torch.empty_like(send)
    hrecv = torch.empty_like(hsend)
    comm.all_to_all([send], [recv])
    comm.halo([hsend], [hrecv])
    rs, rm = red.clone(), red.clone()
    comm.allreduce([rs], SUM)
    comm.allreduce([rm], MAX)
    q.put((rank, recv.numpy(), hrecv.numpy(), rs.numpy(), rm.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_slab_exchanges_match_in_process_emulation(world):
    # DistComm (one process per rank) moves exactly what LocalComm (the single-GPU emulation
    # the GPU parity tests run) moves: all-to-all blocks, periodic halo planes, reductions.
    import numpy as np

    from paper_2508_02681_b200.slab import MAX, SUM, LocalComm

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    loc = LocalComm(world)
    bufs = [_slab_bufs(r, world) for r in range(world)]
    sends = [b[0] for b in bufs]
    recvs = [s.clone() * 0 for s in sends]
    loc.all_to_all(sends, recvs)
    hs = [b[1] for b in bufs]
    hr = [h.clone() * 0 for h in hs]
    loc.halo(hs, hr)
    rs = [b[2].clone() for b in bufs]
    rm = [b[2].clone() for b in bufs]
    loc.allreduce(rs, SUM)
    loc.allreduce(rm, MAX)
    for rank, recv, hrecv, s, m in outs:
        np.testing.assert_array_equal(recv, recvs[rank].numpy())
        np.testing.assert_array_equal(hrecv, hr[rank].numpy())
        np.testing.assert_allclose(s, rs[rank].numpy(), rtol=1e-15)
        np.testing.assert_array_equal(m, rm[rank].numpy())
    # the all-to-all is a block transpose; the halo delivers each rank its z-neighbours' planes
    for q_ in range(world):
        for r in range(world):
            np.testing.assert_array_equal(recvs[q_][r].numpy(), sends[r][q_].numpy())
        np.testing.assert_array_equal(hr[q_][0].numpy(), hs[(q_ - 1) % world][1].numpy())
        np.testing.assert_array_equal(hr[q_][1].numpy(), hs[(q_ + 1) % world][0].numpy())
