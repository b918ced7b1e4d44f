#!/usr/bin/env python
"""UNO-CG hot-path benchmark (BASELINE.json metric: PCG DOF-iterations/s at 256^3).

One *step* = the whole hot path over the fixed config-3 batch: 48
problems (8 Boolean-sphere microstructures at vf 0.1..0.4 x contrasts {2,5,10,20,50,100},
256^3 thermal, periodic), sharded over the ranks (Latin square at 8 GPUs, LPT on
the Eq 27 cost at 2/4; no data-path collective).  For each of its problems a rank re-targets its
solver (reference medium, tabulated G_hat, Eq 55 check), solves the 3 load cases with Alg 2 to
rel. ||r||_inf 1e-8, removes the mean and computes the effective conductivity.
value = sum over ranks/solves of (DOF x iterations) / max-over-ranks device time (strong
scaling: the batch is fixed; --weak gives every rank its own 48-problem batch instead).

Launch: python bench.py --gpus N --steps K --warmup W   (N > 1 under torchrun, NCCL).
        python bench.py --impl reference ...              (the CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG DOF-iterations/s at 256³ (1/2/4/8 B200); K·p & UNO-apply HBM GB/s vs peak"
UNIT = "DOF-iterations/s"
N_GRID = 256
CONTRASTS = (2.0, 5.0, 10.0, 20.0, 50.0, 100.0)
N_MICRO = 8
TOL = 1e-8
MAX_IT = 1000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=N_GRID, help="grid edge (256 = config 3; smaller only for debugging)")
    ap.add_argument("--weak", action="store_true", help="every rank solves its own 48-problem batch (weak scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--problems", type=int, default=0,
                    help="profiling only: the first P problems of this rank's shard (0 = all; not a bench value)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def problem_list(ws: int, rank: int, weak: bool):
    """This rank's (microstructure, contrast) problems: its shard of the fixed 48-problem batch
    (dist.config3_shard), or with --weak the whole batch (own microstructure seeds per rank)."""
    from paper_2508_02681_b200 import dist as D

    if weak:
        return D.config3_problems(CONTRASTS, N_MICRO)
    return D.config3_shard(ws, rank, CONTRASTS, N_MICRO)


def make_microstructures(ms, n: int, seed_base: int):
    from paper_2508_02681_b200 import synth

    return {m: synth.config3_microstructure(m, n=n, seed_base=seed_base) for m in sorted(ms)}


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                s, m = float(r[0]), float(r[1])
            except Exception:
                continue
            sm.append(s)
            mx = max(mx, m)
            for k, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- algorithmic bytes
def kernel_bytes(n: int, N1: int, nrhs: int):
    """Algorithmic HBM bytes per launch of each kernel class, thermal c = 1.
    spectrum bytes: 16 B per complex bin, H1/N1 = (N1/2+1)/N1 bins per DOF."""
    spec = 16.0 * (N1 // 2 + 1) / N1  # bytes per DOF of one pass over the half spectrum
    per_dof = {
        "K": 8 + 8 + 1,                  # read d, write p, read phase (1 B/voxel)
        "xfwd": 8 + 8 + 8 + spec,         # read r, p; write r; write r_hat
        "ypass": 2 * spec,               # read + write spectrum (per launch; 2 launches/iter)
        "gpass": 2 * spec + spec / 2,    # read + write spectrum + 8 B G_hat per bin
        "xinv": spec + 8 * 3.5,          # read s_hat; paired u updates (3D handles): odd iterations
                                         # read d_old, write d (16 B), even ones read d_old, d_{j-2},
                                         # u, write d, u (40 B): 28 B/DOF on average
    }
    return {k: v * n * nrhs for k, v in per_dof.items()}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)  # forces communicator creation; logged so the driver can check the ranks
        torch.cuda.synchronize()
        nv = ".".join(str(x) for x in torch.cuda.nccl.version())
        print(f"[bench rank {rank}/{ws}] NCCL {nv} communicator ready on cuda:{local} "
              f"({torch.cuda.get_device_name(local)}), all_reduce check {int(t.item())} == {ws}",
              file=sys.stderr, flush=True)
    from paper_2508_02681_b200 import dist as D
    from paper_2508_02681_b200.api import UnoCG

    n = args.grid
    t0 = time.time()
    probs = problem_list(ws, rank, args.weak)
    if args.problems > 0:
        probs = probs[:args.problems]
    seed_base = 300 + 8 * rank if args.weak else 300
    micro = make_microstructures({m for m, _ in probs}, n, seed_base)
    phases = {m: torch.from_numpy(v).to(dev) for m, v in micro.items()}
    loads = np.eye(3)
    u = torch.empty((3, 1, n, n, n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    gen_s = time.time() - t0
    # one solver per rank: its workspace is allocated once (like model memory); every problem
    # of a step re-runs the a0 setup (reference medium, G_hat table, Eq 55) via uno_cg_update.
    m0, R0 = probs[0]
    solver = UnoCG(phases[m0], "thermal", (1.0, R0), nrhs=3, seed=3000 + m0, amp=0.1, stream=stream)

    def one_step(timing: bool, pev=None):
        dofit = 0
        launches = 0
        kt = {}
        effs = []
        s = solver
        for i, (m, R) in enumerate(probs):
            if pev is not None:
                pev[i][0].record(stream)
            s.update(phases[m], (1.0, R), seed=3000 + m, amp=0.1)
            launches += 2  # symbol build + Eq 55
            if timing:
                s.kernel_timing(enable=1, reset=1)
            res = s.solve(loads, rel_tol=TOL, max_iter=MAX_IT, out=u)
            launches += res.launches
            dofit += sum(r["iterations"] for r in res.reports) * n ** 3
            effs.append(s.effective_property(res.u, loads))
            launches += 2
            if pev is not None:
                pev[i][1].record(stream)
                pits.append([r["iterations"] for r in res.reports])
            if timing:
                for k, (ms, c) in s.kernel_timing().items():
                    a = kt.setdefault(k, [0.0, 0])
                    a[0] += ms
                    a[1] += c
                s.kernel_timing(enable=0)
        return dofit, launches, kt, effs

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        one_step(False)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # per-problem device time of the first timed step (events between problems: negligible cost)
    pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in probs]
    pits = []
    tot_dofit, tot_launch, ktimes = 0, 0, {}
    with ClockSampler(local) as clk:
        # timed region: the production path (each solve one CUDA graph with a device-side WHILE loop)
        barrier()
        ev0.record(stream)
        for k_ in range(args.steps):
            d_, l_, _, effs = one_step(False, pev if k_ == 0 else None)
            tot_dofit += d_
            tot_launch += l_
        ev1.record(stream)
        barrier()
        # kernel-timing region: the same steps again with a CUDA-event pair around every kernel
        # launch (chunked graphs; the event nodes cost ~10 % of the step, so it is kept out of
        # `value`).  Per-kernel durations for the roofline come from here.
        kt0, kt1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        kt0.record(stream)
        kt_dofit = 0
        for _ in range(args.steps):
            d_, _, kt, _ = one_step(True)
            kt_dofit += d_
            for k, (ms_, c) in kt.items():
                a = ktimes.setdefault(k, [0.0, 0])
                a[0] += ms_
                a[1] += c
        kt1.record(stream)
        barrier()
    my_ms = ev0.elapsed_time(ev1)
    prob_ms = [round(a.elapsed_time(b), 2) for a, b in pev]
    ms = D.reduce_max(my_ms)                      # max over ranks of the device time
    rank_ms = D.gather_results([my_ms])
    all_dofit = D.reduce_sum(float(tot_dofit))    # units processed by all ranks
    value = all_dofit / (ms / 1e3)
    kt_ms = D.reduce_max(kt0.elapsed_time(kt1))
    kt_value = D.reduce_sum(float(kt_dofit)) / (kt_ms / 1e3)

    # ---- roofline of the dominant kernel (live per-launch CUDA-event durations) ----
    peak, peak_src = peaks()
    kb = kernel_bytes(n ** 3, n, 3)
    per = {}
    for k, (kms, cnt) in ktimes.items():
        if cnt and k in kb:
            avg_ms = kms / cnt
            per[k] = {"avg_us": avg_ms * 1e3, "launches": cnt, "share": kms, "GBps": kb[k] / (avg_ms / 1e3) / 1e9}
    tot_k = sum(v["share"] for v in per.values()) or 1.0
    for v in per.values():
        v["share"] = v["share"] / tot_k
    dom = max(per, key=lambda k: per[k]["share"]) if per else None
    roof = None
    if dom:
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic_r02.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(per[dom]["GBps"], 1), "peak": peak, "unit": "GB/s",
                "frac": round(per[dom]["GBps"] / peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": kb[dom], "peak_source": peak_src,
                "timing": "CUDA-event pairs around every launch on the launch stream, in a second timed pass of "
                          f"the same {args.steps} steps (that pass ran at {kt_value / 1e9:.2f} G{UNIT})",
                "kernels": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in per.items()}}

    # ---- whole-iteration roofline (north star: bytes per iteration / HBM peak) ----
    per_it = {"K": 1, "xfwd": 1, "ypass": 2, "gpass": 1, "xinv": 1}
    b_dof_it = sum(kb[k] * c for k, c in per_it.items()) / (n ** 3 * 3)
    iter_roof = {"bytes_per_dof_iteration": round(b_dof_it, 2),
                 "achieved_GBps": round(value * b_dof_it / 1e9, 1),
                 "frac_measured_peak": round(value * b_dof_it / 1e9 / peak, 4),
                 "frac_nominal_8TBs": round(value * b_dof_it / 8e12, 4),
                 "note": "5-pass schedule algorithmic bytes (DESIGN.md §5) x DOF-iterations/s of `value` "
                         "(includes the per-problem setup inside the step)"}

    # ---- e2e: host buffers in, host results out, through the public API ----
    e2e = None
    if not args.no_e2e:
        host_ph = {m: torch.from_numpy(v).pin_memory() for m, v in micro.items()}
        dph = {m: torch.empty_like(p, device=dev) for m, p in host_ph.items()}
        h2d = sum(p.numel() for p in host_ph.values())
        d2h = 0

        def e2e_step():
            nonlocal d2h
            d2h = 0
            dofit = 0
            for m, p in host_ph.items():
                dph[m].copy_(p, non_blocking=True)
            out = []
            s = solver
            for (m, R) in probs:
                s.update(dph[m], (1.0, R), seed=3000 + m, amp=0.1)
                res = s.solve(loads, rel_tol=TOL, max_iter=MAX_IT, out=u)
                keff = s.effective_property(res.u, loads)  # device -> host (9 doubles)
                out.append((keff, [r["iterations"] for r in res.reports]))
                d2h += keff.nbytes + 3 * 40  # kappa_bar + per-load reports
                dofit += sum(r["iterations"] for r in res.reports) * n ** 3
            return dofit

        e2e_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dsum = 0
        for _ in range(args.steps):
            dsum += e2e_step()
        e1.record(stream)
        barrier()
        ems = D.reduce_max(e0.elapsed_time(e1))
        dsum = D.reduce_sum(float(dsum))
        e2e = {"value": dsum / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:  # the oracle baseline is an N = 1 figure
        cpu = cpu_baseline(n)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg3: fixed batch of 48 problems (8 Boolean-sphere microstructures vf 0.1-0.4 x "
                                   f"6 contrasts 2-100) x 3 loads, {n}^3 thermal periodic Q1, rel ||r||_inf 1e-8"
                                   + (" (--weak: 48 per rank)" if args.weak else f", sharded over {ws} rank(s)"),
                       "global_batch": 48 * ws if args.weak else 48, "grid": n, "loads": 3, "dof_per_solve": n ** 3,
                       "l2": "inputs larger than L2 (~1.7 GB working set per solve vs 126 MB L2)",
                       "parallelism": (f"batch-shard x{ws}: " + ("Latin square" if ws == 8 else "LPT on Eq 27 cost"
                                                                  if ws > 1 else "single GPU")
                                       + " (no data-path collective)"),
                       "problems_per_rank": len(probs),
                       "rank_ms": [round(x, 1) for x in rank_ms],
                       "imbalance_max_over_mean": round(max(rank_ms) / (sum(rank_ms) / len(rank_ms)), 4),
                       "problems": [f"m{m}R{R:g}" for m, R in probs] if ws == 1 else None,
                       "problem_ms_step1": prob_ms if ws == 1 else None,
                       "problem_iterations": pits if ws == 1 else None,
                       "input_generation_s": round(gen_s, 1)},
            "roofline": roof, "iteration_roofline": iter_roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(tot_launch),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- CPU oracle
def _host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class _OracleSample:
    """The CPU oracle on one config-3 problem (microstructure 3, R = 20, seed 3003) and load e_1:
    Alg 2 with the oracle's K (fem.apply_K_chunked: threads over z-slabs) and UNO apply (scipy.fft
    with `workers`), on the box's host cores.  Setup (G_hat, f) is outside the
    timer; `run(k)` times k PCG iterations and returns (DOF-iterations, seconds)."""

    def __init__(self, n: int):
        from oracle import fem, greens, transform
        from paper_2508_02681_b200 import synth

        self.cores = _host_cores()
        self.n = n
        self.zchunk = max(4, -(-n // self.cores))
        self.threads = min(self.cores, -(-n // self.zchunk))
        transform.set_workers(self.cores)
        self.phase = synth.config3_microstructure(3, n=n)
        self.g = fem.Grid((n, n, n), h=1.0 / n)
        self.mat = (1.0, 20.0)
        self.G = greens.ghat(self.g, "thermal", self.mat, 3003, 0.1, half=True)
        self.f = fem.rhs(self.g, "thermal", self.phase, self.mat, np.eye(3)[0])

    def run(self, iters: int):
        from oracle import fem, greens, pcg

        t = time.perf_counter()
        pcg.pcg(lambda v: fem.apply_K_chunked(self.g, "thermal", self.phase, self.mat, v, zchunk=self.zchunk,
                                              workers=self.threads),
                lambda v: greens.apply_precond(self.G, v), self.f, fixed_iters=iters)
        return self.n ** 3 * iters, time.perf_counter() - t

    def describe(self, iters: int, secs: float) -> str:
        return (f"1 problem (ms 3, R=20), 1 load, {iters} PCG iteration(s) at {self.n}^3: oracle K over "
                f"{self.threads} z-slab threads, scipy.fft workers={self.cores}; {secs:.1f} s")


def cpu_baseline(n, target_s: float = 15.0):
    o = _OracleSample(n)
    d1, t1 = o.run(1)
    k = int(min(20, max(1, round(target_s / max(t1, 1e-3)))))
    dofit, dt = o.run(k)
    return {"value": dofit / dt, "unit": UNIT, "cores": o.cores, "threads": o.threads, "kind": "oracle",
            "sample": o.describe(k, dt)}


def run_reference(args):
    """The CPU oracle arm (tier reading of the reference arm): the oracle as it stands on the box's
    host cores, each step a bounded sample of the config-3 workload (2 PCG iterations of one
    problem/load at 256^3), same metric/unit as our arm.  Rank 0 only."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    n = args.grid
    o = _OracleSample(n)
    for _ in range(args.warmup):
        o.run(1)
    tot, tsum = 0, 0.0
    for _ in range(args.steps):
        d, t = o.run(2)
        tot += d
        tsum += t
    value = tot / tsum
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tsum / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"cfg3 sample: 1 problem (ms 3, R=20), 1 load, 2 PCG iterations per step at {n}^3 "
                                   "(CPU oracle; bounded sample of the config-3 workload)", "grid": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": o.cores, "threads": o.threads, "kind": "oracle",
                             "sample": o.describe(2, tsum / max(args.steps, 1)) + " per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
