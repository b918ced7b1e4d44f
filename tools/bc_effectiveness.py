"""DESIGN.md §7b table: one config-3 problem (256^3 thermal, Boolean spheres j = 3, kappa 1/20,
3 loads) solved to rel ||r||_inf <= 1e-8 with UNO-CG and Jacobi-CG for the periodic, mixed
(Dirichlet z) and all-Dirichlet boundaries: iterations per load and device time per iteration."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

ph = torch.from_numpy(synth.config3_microstructure(3)).cuda()
print(f"{'BC':22s} {'precond':8s} {'iterations':>18s} {'us/iteration':>13s}")
for name, bc in [("periodic", (0, 0, 0)), ("mixed (Dirichlet z)", (0, 0, 1)), ("all Dirichlet", (1, 1, 1))]:
    for pc in ("uno", "jacobi"):
        s = UnoCG(ph, "thermal", (1.0, 20.0), nrhs=3, seed=3003, amp=0.1, bc=bc, precond=pc)
        s.solve(np.eye(3), rel_tol=1e-8, max_iter=5000)  # warm-up (graph build)
        r = s.solve(np.eye(3), rel_tol=1e-8, max_iter=5000)
        its = [rep["iterations"] for rep in r.reports]
        print(f"{name:22s} {pc:8s} {' / '.join(map(str, its)):>18s} {1e3 * r.ms / max(its):13.0f}")
        s.close()
