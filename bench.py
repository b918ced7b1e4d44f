#!/usr/bin/env python
"""UNO-CG hot-path benchmark (BASELINE.json metric: PCG DOF-iterations/s at 256^3).

One *step* = the whole hot path over one batch of synthetic
config-3 input: for each of the rank's 48 problems (8 Boolean-sphere microstructures at
vf 0.1..0.4 x contrasts {2,5,10,20,50,100}, 256^3 thermal, periodic) create the solver
(reference medium, tabulated G_hat, Eq 55 check), solve its 3 load cases with Alg 2 to
rel. ||r||_inf 1e-8, remove the mean and compute the effective conductivity.
value = sum over ranks/solves of (DOF x iterations) / max-over-ranks device time.

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
    ap.add_argument("--problems", type=int, default=48, help="problems per rank (48 = config 3)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def problem_list(rank: int, nprob: int):
    """Rank-local problems (weak scaling): microstructure m of this rank x contrast j."""
    out = []
    for i in range(nprob):
        m, j = i % N_MICRO, (i // N_MICRO) % len(CONTRASTS)
        out.append((m, CONTRASTS[j]))
    return out


def make_microstructures(rank: int, n: int):
    from paper_2508_02681_b200 import synth

    return [synth.config3_microstructure(j, n=n, seed_base=300 + 8 * rank) for j in range(N_MICRO)]


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
        "xinv": spec + 8 * 4,            # read s_hat; read d, u; write d, u
    }
    return {k: v * n * nrhs for k, v in per_dof.items()}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2508_02681_b200 import dist as D
    from paper_2508_02681_b200.api import UnoCG

    n = args.grid
    t0 = time.time()
    micro = make_microstructures(rank, n)
    probs = problem_list(rank, args.problems)
    phases = [torch.from_numpy(m).to(dev) for m in micro]
    loads = np.eye(3)
    u = torch.empty((3, 1, n, n, n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    gen_s = time.time() - t0
    # one solver per rank: its workspace is allocated once (like model memory); every problem
    # of a step re-runs the a0 setup (reference medium, G_hat table, Eq 55) via uno_cg_update.
    solver = UnoCG(phases[0], "thermal", (1.0, CONTRASTS[0]), nrhs=3, seed=3000, amp=0.1, stream=stream)

    def one_step(timing: bool):
        dofit = 0
        launches = 0
        kt = {}
        effs = []
        s = solver
        for (m, R) in probs:
            s.update(phases[m], (1.0, R), seed=3000 + m, amp=0.1)
            launches += 2  # symbol build + Eq 55
            if timing:
                s.kernel_timing(enable=1, reset=1)
            res = s.solve(loads, rel_tol=TOL, max_iter=MAX_IT, out=u)
            launches += res.launches
            dofit += sum(r["iterations"] for r in res.reports) * n ** 3
            effs.append(s.effective_property(res.u, loads))
            launches += 2
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
    tot_dofit, tot_launch, ktimes = 0, 0, {}
    with ClockSampler(local) as clk:
        # timed region: the production path (each solve one CUDA graph with a device-side WHILE loop)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            d_, l_, _, effs = one_step(False)
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
    ms = D.reduce_max(ev0.elapsed_time(ev1))      # max over ranks of the device time
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
        tf = os.path.join(ROOT, "profiles", "traffic_r01.json")
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
        host_ph = [torch.from_numpy(m).pin_memory() for m in micro]
        dph = [torch.empty_like(p, device=dev) for p in host_ph]
        h2d = sum(p.numel() for p in host_ph)
        d2h = 0

        def e2e_step():
            nonlocal d2h
            d2h = 0
            dofit = 0
            for i, p in enumerate(host_ph):
                dph[i].copy_(p, non_blocking=True)
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
        cpu = cpu_baseline(micro[3], 20.0, n)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg3: {args.problems} problems/rank (8 Boolean-sphere microstructures vf 0.1-0.4 x "
                                   f"6 contrasts 2-100) x 3 loads, {n}^3 thermal periodic Q1, rel ||r||_inf 1e-8",
                       "global_batch": args.problems * ws, "grid": n, "loads": 3, "dof_per_solve": n ** 3,
                       "l2": "inputs larger than L2 (~1.7 GB working set per solve vs 126 MB L2)",
                       "parallelism": f"batch-shard x{ws} (no data-path collective)",
                       "input_generation_s": round(gen_s, 1)},
            "roofline": roof, "iteration_roofline": iter_roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(tot_launch),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- CPU oracle
def _oracle_sample(phase, R, n, iters):
    """One load case of one config-3 problem, `iters` PCG iterations with the oracle (setup
    outside the timer).  Returns (DOF-iterations, seconds)."""
    from oracle import fem, greens, pcg

    g = fem.Grid((n, n, n), h=1.0 / n)
    mat = (1.0, R)
    G = greens.ghat(g, "thermal", mat, 3003, 0.1)
    f = fem.rhs(g, "thermal", phase, mat, np.eye(3)[0])
    t = time.perf_counter()
    pcg.pcg(lambda v: fem.apply_K(g, "thermal", phase, mat, v), lambda v: greens.apply_precond(G, v), f,
            fixed_iters=iters)
    dt = time.perf_counter() - t
    return n ** 3 * iters, dt


def cpu_baseline(phase, R, n, iters=2):
    dofit, dt = _oracle_sample(phase, R, n, iters)
    return {"value": dofit / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"1 problem (ms 3, R={R:g}), 1 load, {iters} PCG iterations at {n}^3, NumPy single thread; "
                      f"{dt:.1f} s"}


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    n = args.grid
    from paper_2508_02681_b200 import synth

    phase = synth.config3_microstructure(3, n=n)
    for _ in range(args.warmup):
        _oracle_sample(phase, 20.0, n, 1)
    tot, tsum = 0, 0.0
    for _ in range(args.steps):
        d, t = _oracle_sample(phase, 20.0, n, 1)
        tot += d
        tsum += t
    value = tot / tsum
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tsum / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"cfg3 sample: 1 problem (ms 3, R=20), 1 load, 1 PCG iteration per step at {n}^3 "
                                   "(CPU oracle; bounded sample of the config-3 workload)", "grid": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": "1 load x 1 iteration per step at 256^3, NumPy single thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
