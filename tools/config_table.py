"""Per-config throughput on one GPU through the production path (CUDA-graph WHILE loop):
configs 0-2 of BASELINE.json at their own sizes (all loads of the config in one handle), config 3
one problem (the bench runs 48), config 4 periodic and mixed with one load.  Iterations to
rel ||r||_inf <= 1e-8 (config 4: 20 fixed iterations), device time per iteration, DOF-it/s."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402


def run(name, phase, physics, mat, loads, seed, amp, bc=None, fixed=0):
    ph = torch.from_numpy(phase).cuda()
    kw = {"bc": bc} if bc else {}
    s = UnoCG(ph, physics, mat, nrhs=len(loads), seed=seed, amp=amp, **kw)
    s.solve(loads, rel_tol=1e-8, max_iter=2000, fixed_iters=fixed)  # warm-up (graph build)
    r = s.solve(loads, rel_tol=1e-8, max_iter=2000, fixed_iters=fixed)
    its = [rep["iterations"] for rep in r.reports]
    dof = int(np.prod(phase.shape)) * (1 if physics == "thermal" else phase.ndim)
    if bc and bc[-1] == 1 and phase.ndim == 3:
        dof = dof * (phase.shape[0] - 1) // phase.shape[0]
    us = 1e3 * r.ms / max(its)
    gdofit = dof * sum(its) / (r.ms * 1e-3) / 1e9
    print(f"{name:34s} {len(loads):3d} {str(its):>24s} {us:10.1f} {gdofit:9.2f}", flush=True)
    s.close()


print(f"{'config':34s} {'nrhs':>3s} {'iterations':>24s} {'us/iter':>10s} {'GDOF-it/s':>9s}")
for P in (synth.config0(), synth.config1(), synth.config2()):
    run(P.name, P.phase, P.physics, P.mat, P.loads, P.seed, P.amp)
ph3 = synth.config3_microstructure(3)
run("cfg3 one problem (256^3, R=20)", ph3, "thermal", (1.0, 20.0), np.eye(3), 3003, 0.1)
P4 = synth.config4()
run("cfg4 512^3 elastic periodic", P4.phase, "elastic", P4.mat, P4.loads[:1], P4.seed, P4.amp, fixed=20)
run("cfg4 512^3 elastic mixed (Dir. z)", P4.phase, "elastic", P4.mat, P4.loads[:1], P4.seed, P4.amp, bc=(0, 0, 1), fixed=20)
