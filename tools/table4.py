"""PAPER.md Tab 4 on a config-1 problem (64^3 thermal, RSA spheres vf 0.3, contrast
100, load e1) with the library: per preconditioner the PCG iterations to rel. ||r||_inf <= tol and
the Lanczos estimates of lambda_min / lambda_max / cond_2 / C_CG / N_iter_est (uno_cg_spectrum),
effectiveness = N_iter(CG) / N_iter(P)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tol", type=float, default=1e-6)
a = ap.parse_args()
P = synth.config1()
ph = torch.from_numpy(P.phase).cuda()
rows = []
for name, precond, seed, amp in [("CG (P = I)", "identity", P.seed, P.amp), ("Jac-CG", "jacobi", P.seed, P.amp),
                                 ("UNO-CG (perturbed FANS, R6)", "uno", P.seed, P.amp), ("FANS", "uno", 0, 0.0)]:
    s = UnoCG(ph, "thermal", P.mat, nrhs=1, seed=seed, amp=amp, precond=precond)
    r = s.solve(np.eye(3)[:1], rel_tol=a.tol, max_iter=20000)
    sp = s.spectrum(0, tol=a.tol)
    rows.append((name, r.reports[0]["iterations"], sp))
    s.close()
n_cg = rows[0][1]
print(f"config 1: 64^3 thermal, kappa {P.mat}, load e1, rel ||r||_inf <= {a.tol:g}")
print(f"{'solver':30s} {'lambda_max':>10s} {'lambda_min':>10s} {'cond_2':>12s} {'C_CG':>7s} {'N_est':>8s} {'N_iter':>7s} {'effect.':>8s}")
for name, its, sp in rows:
    print(f"{name:30s} {sp['lambda_max']:10.4f} {sp['lambda_min']:10.6f} {sp['cond']:12.4f} {sp['C_CG']:7.4f} "
          f"{sp['N_iter_est']:8.1f} {its:7d} {n_cg / its:8.1f}")
