"""Small solves through every kernel family, for `compute-sanitizer --tool memcheck` (one tool per
run): periodic thermal / elastic (3D, 2D), mixed (Dirichlet z), all-Dirichlet, the one-CTA 2D
solve, the baseline preconditioners, apply_K / apply_precond / rhs / effective property, the
256-point register-direct passes (N2 = N3 = 256 with a short x axis) and emulated slab ranks."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402
from paper_2508_02681_b200.slab import LocalComm, SlabSolver  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
el = (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(10.0, 0.2))
cases = [((32, 16, 8), "thermal", (0, 0, 0)), ((16, 16, 8), "elastic", (0, 0, 0)), ((32, 32), "thermal", (0, 0)),
         ((16, 16), "elastic", (0, 0)), ((32, 16, 16), "thermal", (0, 0, 1)), ((16, 16, 8), "elastic", (0, 0, 1)),
         ((32, 16, 16), "thermal", (1, 1, 1)), ((32, 32), "thermal", (0, 1)), ((8, 256, 256), "thermal", (0, 0, 0)),
         ((256, 16, 16), "thermal", (0, 0, 0)), ((16, 16, 256), "elastic", (0, 0, 0))]
for N, phys, bc in cases:
    ph = torch.from_numpy((rng.random(tuple(reversed(N))) < 0.3).astype(np.uint8)).to(dev)
    mat = (1.0, 10.0) if phys == "thermal" else el
    d = len(N)
    nv = d if phys == "thermal" else d * (d + 1) // 2
    L = np.eye(nv)[:2]
    s = UnoCG(ph, phys, mat, nrhs=2, seed=7, amp=0.1 if phys == "thermal" else 0.05, bc=bc)
    r = s.solve(L, rel_tol=1e-8, max_iter=200)
    s.effective_property(r.u, L)
    v = torch.randn(s.field_shape, dtype=torch.float64, device=dev)
    s.apply_K(v)
    s.apply_precond(v)
    s.kernel_timing(enable=1, reset=1)
    s.solve(L, fixed_iters=3)
    s.kernel_timing(enable=0)
    if bc == (0, 0, 0) and d == 3 and N[0] <= 32:
        for kind in ("jacobi", "identity"):
            s.set_preconditioner(kind)
            s.solve(L, fixed_iters=3)
        s.set_preconditioner("uno")
    s.close()
    print("ok", N, phys, bc, [x["iterations"] for x in r.reports], flush=True)
ph = torch.from_numpy((rng.random((16, 16, 32)) < 0.3).astype(np.uint8)).to(dev)
for peer in (False, True):
    sv = SlabSolver(ph, "thermal", (1.0, 10.0), LocalComm(2), nrhs=1, seed=7, amp=0.1, peer=peer)
    sv.solve(np.eye(3)[:1], fixed_iters=4)
    print("ok slab peer" if peer else "ok slab a2a", flush=True)
torch.cuda.synchronize()
print("sanitize_small done")
