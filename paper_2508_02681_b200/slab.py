"""z-slab decomposition of one UNO-CG problem over several ranks (include/uno_cg_slab.h;
SURVEY.md §8(e) "Config 4 (one 512^3 grid)").

Orchestration only: every arithmetic step of PAPER.md Alg 2 runs in libunocg kernels
(binding.uno_slab_*); this module allocates the exchange buffers, moves them between ranks
and sequences the stages of one iteration:

    forward -> [||r|| all-reduce] -> all-to-all -> green -> [gamma all-reduce] -> all-to-all
    -> inverse -> halo exchange -> kapply -> [d.p all-reduce]

Three transports implement the exchanges with identical buffer semantics:
  * DistComm  — one rank per process/GPU, torch.distributed (NCCL on GPUs; gloo in the CPU
                tests), point-to-point batches for the all-to-all and the halo planes; the
                peer-memory receive buffers live in torch symmetric memory;
  * IpcComm   — one rank per process, receive buffers exported with CUDA IPC handles (every
                rank maps every peer's buffer; the library's pack kernels store straight into
                them), scalars and stage ordering over a torch.distributed group (gloo or
                NCCL) with a stream synchronisation per stage: no kernel ever waits on another
                process, so it also runs two ranks on ONE GPU (the multi-process test);
  * LocalComm — all ranks emulated in this process (one device), plain copies.  Used by the
                single-GPU parity tests: the per-rank kernels and the data movement pattern
                are exactly those of the multi-GPU run.

The iteration loop checks convergence on the host only once per chunk of `check_every`
iterations (converged loads freeze themselves on the device, so the extra bodies are no-ops);
with graph=True the chunk is captured once as a CUDA graph (exchanges included) and replayed.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import binding as B

SUM, MAX = "sum", "max"


class LocalComm:
    """All `nranks` ranks live in this process; buffers are lists indexed by rank."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.ranks = list(range(nranks))

    def all_to_all(self, sends, recvs):
        # recvs[q][r] <- sends[r][q]  (block r of rank q's receive buffer came from rank r)
        for r in self.ranks:
            for q in self.ranks:
                recvs[q][r].copy_(sends[r][q])

    def halo(self, sends, recvs):
        # sends[r][0] = first node plane of rank r -> rank r-1 (its plane zlo+Z)
        # sends[r][1] = last node plane of rank r  -> rank r+1 (its plane zlo-1)
        n = self.nranks
        for r in self.ranks:
            recvs[(r - 1) % n][1].copy_(sends[r][0])
            recvs[(r + 1) % n][0].copy_(sends[r][1])

    def peer_buffers(self, numel: int, device):
        """Receive buffers for the peer-memory exchange: one per rank, each rank's pointer list
        holds every rank's buffer (all in this process).  Returns (buffers, pointer lists, token)."""
        bufs = [torch.empty(numel, dtype=torch.float64, device=device) for _ in self.ranks]
        ptrs = [[b.data_ptr() for b in bufs] for _ in self.ranks]
        return bufs, ptrs, None

    def peer_barrier(self, token):
        pass  # one stream: the emulated ranks' kernels are already ordered

    def allreduce(self, vals, op: str):
        tot = vals[0].clone()
        for v in vals[1:]:
            tot = tot + v if op == SUM else torch.maximum(tot, v)
        for v in vals:
            v.copy_(tot)


class DistComm:
    """One rank per process (torch.distributed already initialised)."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.nranks = dist.get_world_size()
        self.ranks = [self.rank]

    def all_to_all(self, sends, recvs):
        send, recv = sends[0], recvs[0]
        r, n = self.rank, self.nranks
        recv[r].copy_(send[r])
        ops = []
        for k in range(1, n):  # pairwise order: every rank sends to r+k while receiving from r-k
            q_to, q_from = (r + k) % n, (r - k) % n
            ops.append(self.dist.P2POp(self.dist.isend, send[q_to], q_to))
            ops.append(self.dist.P2POp(self.dist.irecv, recv[q_from], q_from))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def halo(self, sends, recvs):
        send, recv = sends[0], recvs[0]
        r, n = self.rank, self.nranks
        if n == 1:
            recv[1].copy_(send[0])
            recv[0].copy_(send[1])
            return
        lo, hi = (r - 1) % n, (r + 1) % n
        ops = [self.dist.P2POp(self.dist.isend, send[0], lo), self.dist.P2POp(self.dist.irecv, recv[1], hi),
               self.dist.P2POp(self.dist.isend, send[1], hi), self.dist.P2POp(self.dist.irecv, recv[0], lo)]
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()

    def peer_buffers(self, numel: int, device):
        """Receive buffers in symmetric memory (torch.distributed._symmetric_memory): every rank's
        buffer is mapped into every process over NVLink; `buffer_ptrs` are the peer addresses.
        The rendezvous handle is the token its barrier is taken on (one per buffer / solver)."""
        import torch.distributed._symmetric_memory as symm_mem

        buf = symm_mem.empty(numel, dtype=torch.float64, device=device)
        hdl = symm_mem.rendezvous(buf, self.dist.group.WORLD)
        return [buf], [list(hdl.buffer_ptrs)], hdl

    def peer_barrier(self, token):
        # device-side barrier over the symmetric-memory signal pads (stream-ordered on the current
        # stream, which SlabSolver makes the library's stream): every rank's peer stores of the
        # stage have landed before anyone reads its receive buffer
        token.barrier()

    def allreduce(self, vals, op: str):
        self.dist.all_reduce(vals[0], op=self.dist.ReduceOp.SUM if op == SUM else self.dist.ReduceOp.MAX)


class IpcComm:
    """One rank per process; peer receive buffers shared with CUDA IPC handles, control over a
    torch.distributed group (gloo in the single-GPU multi-process test).  A stage's peer stores
    are ordered before the peers' reads by a stream synchronisation and a group barrier on the
    host (peer_barrier), never by a kernel waiting on another process."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.ranks = [self.rank]
        self._keep = []  # peers' mapped storages stay alive with the communicator

    def _cpu(self, x):
        return x.detach().to("cpu")

    def peer_buffers(self, numel: int, device):
        from torch.multiprocessing.reductions import reduce_tensor

        buf = torch.zeros(numel, dtype=torch.float64, device=device)
        torch.cuda.synchronize()
        mine = reduce_tensor(buf)  # (rebuild function, args): a picklable CUDA IPC handle
        allh = [None] * self.nranks
        self.dist.all_gather_object(allh, mine, group=self.group)
        ptrs = []
        for q, (fn, args) in enumerate(allh):
            if q == self.rank:
                ptrs.append(buf.data_ptr())
            else:
                t = fn(*args)  # maps rank q's buffer into this process (cudaIpcOpenMemHandle)
                self._keep.append(t)
                ptrs.append(t.data_ptr())
        return [buf], [ptrs], None

    def peer_barrier(self, token):
        torch.cuda.current_stream().synchronize()  # this rank's peer stores are complete
        self.dist.barrier(group=self.group)        # ... and so are everyone else's

    def allreduce(self, vals, op: str):
        t = self._cpu(vals[0])
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM if op == SUM else self.dist.ReduceOp.MAX, group=self.group)
        vals[0].copy_(t)

    def all_to_all(self, sends, recvs):
        raise NotImplementedError("IpcComm carries the peer-memory exchange only (SlabSolver(peer=True))")

    def halo(self, sends, recvs):
        raise NotImplementedError("IpcComm carries the peer-memory exchange only (SlabSolver(peer=True))")


@dataclass
class SlabResult:
    u: list          # per local rank: [nrhs][c][Z][N2][N1] (mean-free per component)
    reports: list    # per load: iterations, converged, status, r0_inf, rel_res, gamma_last
    iterations: int  # loop bodies executed


class SlabSolver:
    """UNO-CG on a z-slab decomposed grid.  `phase` is the whole [N3][N2][N1] uint8 field on
    this process's device (every rank keeps all of it: 1 byte per voxel).  bc = (0, 0, 1): Dirichlet
    faces on z (config 4's mixed variant); vectors then keep N3 node planes with plane 0 (the fixed
    face, rank 0's first plane) held at 0 — the whole-grid handle's planes 1..N3-1."""

    def __init__(self, phase: torch.Tensor, physics: str, mat, comm, nrhs: int = 1, seed: int = 0, amp: float = 0.0,
                 h: float = 0.0, ref=None, peer: bool = False, graph: bool | None = None, bc=(0, 0, 0)):
        """graph: capture a chunk of iterations as one CUDA graph (default: only for LocalComm,
        whose exchanges are device copies; IpcComm orders stages on the host and cannot be)."""
        assert phase.dim() == 3 and phase.dtype == torch.uint8 and phase.is_cuda
        self.phase = phase.contiguous()
        self.comm = comm
        self.nrhs = nrhs
        N3, N2, N1 = self.phase.shape
        self.c = 1 if physics == "thermal" else 3
        d = B.UnoCgDesc()
        d.dim = 3
        d.n[0], d.n[1], d.n[2] = N1, N2, N3
        d.h = h
        d.physics = B.UNO_THERMAL if physics == "thermal" else B.UNO_ELASTIC
        if physics == "thermal":
            d.mat[0][0], d.mat[1][0] = float(mat[0]), float(mat[1])
        else:
            (d.mat[0][0], d.mat[0][1]), (d.mat[1][0], d.mat[1][1]) = mat
        if ref is not None:
            if physics == "thermal":
                d.ref[0] = float(ref)
            else:
                d.ref[0], d.ref[1] = ref
        d.seed, d.amp, d.nrhs = seed, amp, nrhs
        self.bc = tuple(int(b) for b in bc)
        for i, b in enumerate(self.bc):
            d.bc[i] = b
        d.stream = torch.cuda.current_stream().cuda_stream
        self.desc = d
        self.handles = [B.uno_slab_create(d, r, comm.nranks, self.phase) for r in comm.ranks]
        nvec, blk, hs, Z = B.uno_slab_sizes(self.handles[0])
        self.Z, self.shape = Z, (nrhs, self.c, Z, N2, N1)
        dev = self.phase.device
        f64 = dict(dtype=torch.float64, device=dev)
        R = comm.nranks
        self.send = [torch.empty((R, 2 * blk), **f64) for _ in comm.ranks]
        self.recv = [torch.empty((R, 2 * blk), **f64) for _ in comm.ranks]
        self.hsend = [torch.empty((2, hs), **f64) for _ in comm.ranks]
        self.hrecv = [torch.empty((2, hs), **f64) for _ in comm.ranks]
        self.red = [torch.empty(nrhs, **f64) for _ in comm.ranks]
        # peer-memory exchange: the pack kernels store straight into the receivers' buffers (A for
        # the forward transpose, B for the way back); no send buffers, no all-to-all call
        self.peer = peer
        if peer:
            ra, self.ptrA, self.tokA = comm.peer_buffers(R * 2 * blk, dev)
            rb, self.ptrB, self.tokB = comm.peer_buffers(R * 2 * blk, dev)
            self.recvA = [t.view(R, 2 * blk) for t in ra]
            self.recvB = [t.view(R, 2 * blk) for t in rb]
            hr, self.ptrH, self.tokH = comm.peer_buffers(2 * hs, dev)
            self.hrecv = [t.view(2, hs) for t in hr]
        self.graph = isinstance(comm, LocalComm) if graph is None else bool(graph)
        self._graphs = {}

    def close(self):
        for h in self.handles:
            B.uno_slab_destroy(h)
        self.handles = []

    def _scalar(self, slot: int, op: str):
        for h, v in zip(self.handles, self.red):
            B.uno_slab_reduce(h, slot, v)
        self.comm.allreduce(self.red, op)
        for h, v in zip(self.handles, self.red):
            B.uno_slab_apply(h, slot, v)

    def iterate(self):
        """One PCG iteration (Alg 2 l.3-12) on every local rank."""
        c, H = self.comm, self.handles
        if self.peer:
            for h, pa in zip(H, self.ptrA):
                B.uno_slab_forward_peer(h, pa)    # x, y transforms; blocks stored into the peers' A
            c.peer_barrier(self.tokA)
            self._scalar(0, MAX)
            for h, ra, pb in zip(H, self.recvA, self.ptrB):
                B.uno_slab_green_peer(h, ra, pb)  # z . G . z^-1; blocks stored into the peers' B
            c.peer_barrier(self.tokB)
            self._scalar(1, SUM)
            for h, rb, ph in zip(H, self.recvB, self.ptrH):
                B.uno_slab_inverse_peer(h, rb, ph)  # boundary planes into the neighbours' halos
            c.peer_barrier(self.tokH)
            for h, hr in zip(H, self.hrecv):
                B.uno_slab_kapply(h, hr)
            self._scalar(2, SUM)
            return
        for h, s in zip(H, self.send):
            B.uno_slab_forward(h, s)
        self._scalar(0, MAX)                      # ||r||_inf: stop test (l.3)
        c.all_to_all(self.send, self.recv)
        for h, r, s in zip(H, self.recv, self.send):
            B.uno_slab_green(h, r, s)
        self._scalar(1, SUM)                      # gamma_1 = r.s (l.7)
        c.all_to_all(self.send, self.recv)
        for h, r, hs in zip(H, self.recv, self.hsend):
            B.uno_slab_inverse(h, r, hs)
        c.halo(self.hsend, self.hrecv)
        for h, hr in zip(H, self.hrecv):
            B.uno_slab_kapply(h, hr)
        self._scalar(2, SUM)                      # d.p -> alpha (l.10)

    def _use_stream(self):
        st = torch.cuda.current_stream().cuda_stream
        for h in self.handles:
            B.uno_slab_set_stream(h, st)

    def _chunk(self, n: int):
        """n iterations; with graph=True a CUDA graph of them, captured on first use and replayed
        (the handles' launches go to the capture stream while recording)."""
        if not self.graph:
            for _ in range(n):
                self.iterate()
            return
        g = self._graphs.get(n)
        if g is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._use_stream()
                for _ in range(n):
                    self.iterate()
            self._use_stream()  # back to the eager stream
            self._graphs[n] = g
        g.replay()

    def solve(self, loads, rel_tol: float = 1e-8, max_iter: int = 1000, fixed_iters: int = 0,
              check_every: int = 4) -> SlabResult:
        self._use_stream()  # launches follow the caller's current stream
        for h in self.handles:
            B.uno_slab_begin(h, loads, rel_tol, max_iter, fixed_iters)
        cap = (fixed_iters if fixed_iters > 0 else max_iter) + 2
        bodies = 0
        while bodies < cap:
            n = min(check_every, cap - bodies)
            self._chunk(n)
            bodies += n
            active, _ = B.uno_slab_state(self.handles[0], self.nrhs)  # one host sync per chunk
            if not active:
                break
        _, reps = B.uno_slab_state(self.handles[0], self.nrhs)
        us = [torch.empty(self.shape, dtype=torch.float64, device=self.phase.device) for _ in self.handles]
        for h, u in zip(self.handles, us):
            B.uno_slab_finish(h, u)
        if self.bc[2]:  # Dirichlet faces on z: no null space, the fluctuation is not mean-free
            return SlabResult(us, reps, bodies)
        # per-component mean over the whole grid: equal slabs -> mean of the slab means
        means = [torch.empty(self.nrhs * self.c, dtype=torch.float64, device=self.phase.device) for _ in self.handles]
        for h, u, m in zip(self.handles, us, means):
            B.uno_slab_local_means(h, u, m)
        self.comm.allreduce(means, SUM)
        for h, u, m in zip(self.handles, us, means):
            B.uno_slab_subtract_means(h, u, m)
        return SlabResult(us, reps, bodies)
