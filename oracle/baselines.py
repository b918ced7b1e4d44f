"""Baseline preconditioners of PAPER.md §3.2 — oracle (TEST INFRASTRUCTURE ONLY:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm use oracle/).

  P = I        unpreconditioned CG
  P_Jac        the Jacobi preconditioner, Eq 25: (P_Jac)_ii = 1 / A_ii

diag(A) is the sum over the elements touching a node of the element matrices' diagonal
entries (Eq 22), scattered to the nodes exactly as fem.apply_K scatters its element
contributions; the element matrices come from fem's Gauss quadrature.
"""
from __future__ import annotations

import numpy as np

from . import fem, pcg


def diag_K(g: fem.Grid, physics: str, phase: np.ndarray, mat) -> np.ndarray:
    """diag(A) in the field layout (c, free nodes...)."""
    cs = fem.corners(g.d)
    out = fem._pad_full(g, np.zeros(g.field_shape()))
    if physics == "thermal":
        Kref = fem.element_stiffness_thermal(g.d, g.h)
        kap = fem.coeff_field(phase, *mat)[None]
        for ai, a in enumerate(cs):
            fem._scatter_add(g, out, kap * Kref[ai, ai], a)
    else:
        d = g.d
        Kl, Km = fem.element_stiffness_elastic(d, g.h)
        (l0, m0), (l1, m1) = mat
        lam = fem.coeff_field(phase, l0, l1)
        mu = fem.coeff_field(phase, m0, m1)
        for ai, a in enumerate(cs):
            v = np.stack([lam * Kl[d * ai + al, d * ai + al] + mu * Km[d * ai + al, d * ai + al] for al in range(d)])
            fem._scatter_add(g, out, v, a)
    return fem._interior(g, out)


def solve(g: fem.Grid, physics: str, phase, mat, load, kind: str, tol: float = 1e-8, max_iter: int = 10000,
          fixed_iters: int = 0) -> pcg.PCGResult:
    """Alg 1 with P = I ("identity") or P_Jac ("jacobi") from u0 = 0 on the RHS of Eq 76/81."""
    f = fem.rhs(g, physics, phase, mat, load)
    if kind == "identity":
        P = lambda r: r.copy()  # noqa: E731
    elif kind == "jacobi":
        dg = diag_K(g, physics, phase, mat)
        P = lambda r: r / dg  # noqa: E731
    else:
        raise ValueError(kind)
    return pcg.pcg(lambda v: fem.apply_K(g, physics, phase, mat, v), P, f, tol=tol, max_iter=max_iter,
                   fixed_iters=fixed_iters)
