"""Spectral quantities of PAPER.md Tab 4 — oracle (TEST INFRASTRUCTURE ONLY: only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm use oracle/).

Tab 4 reports lambda_max(PA), lambda_min(PA), cond_2(PA), the rate C_CG of Eq 27 and the
bound N_iter,est for each preconditioner.  Two routes, independent of each other:

  dense_spectrum   eigenvalues of the assembled P A (tiny grids; np.linalg.eigvals), without the
                   null space of the periodic problem (the c constant modes);
  ritz_extremes    the Lanczos estimate from the coefficients of Alg 1: CG on P A is a Lanczos
                   process (Saad, Iterative Methods for Sparse Linear Systems, 2nd ed., §6.7.3 — not
                   in the paper), whose m x m tridiagonal built from alpha_j (l.8) and
                   beta_j = gamma_{j+1} / gamma_j (the factor of l.6) is
                       T[j][j]   = 1/alpha_j + beta_{j-1}/alpha_{j-1}      (no second term at j = 0)
                       T[j][j+1] = T[j+1][j] = sqrt(beta_j) / alpha_j ;
                   its eigenvalues are Ritz values of P A, so its extremes approach lambda_min/max
                   from inside as m grows.

cond_2, C_CG and N_iter,est follow from the extremes with pcg.cg_rate / pcg.n_iter_estimate.
"""
from __future__ import annotations

import numpy as np

from . import pcg


def lanczos_T(gamma, alpha) -> np.ndarray:
    """Dense Lanczos tridiagonal of P A from the Alg 1 coefficients gamma_1 and alpha of
    iterations 1..m (lists of equal length m >= 1)."""
    g = np.asarray(gamma, dtype=float)
    a = np.asarray(alpha, dtype=float)
    m = len(a)
    assert m >= 1 and len(g) == m
    T = np.zeros((m, m))
    for j in range(m):
        T[j, j] = 1.0 / a[j]
        if j > 0:
            T[j, j] += (g[j] / g[j - 1]) / a[j - 1]
        if j + 1 < m:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(g[j + 1] / g[j]) / a[j]
    return T


def ritz_extremes(gamma, alpha):
    """(smallest, largest) eigenvalue of lanczos_T."""
    ev = np.linalg.eigvalsh(lanczos_T(gamma, alpha))
    return float(ev[0]), float(ev[-1])


def dense_spectrum(A: np.ndarray, P: np.ndarray, n_null: int) -> np.ndarray:
    """Sorted (real) eigenvalues of P A with the n_null eigenvalues of smallest modulus (the
    constant modes of the periodic problem) removed."""
    ev = np.linalg.eigvals(P @ A)
    assert np.max(np.abs(ev.imag)) < 1e-8 * np.max(np.abs(ev.real))
    ev = ev.real[np.argsort(np.abs(ev.real))][n_null:]
    return np.sort(ev)


def table4_row(lmin: float, lmax: float, tol: float) -> dict:
    """The Tab 4 columns derived from the extreme eigenvalues (Eq 27 with tolerance tol)."""
    cond = lmax / lmin
    return {"lambda_min": lmin, "lambda_max": lmax, "cond": cond, "C_CG": pcg.cg_rate(cond),
            "N_iter_est": pcg.n_iter_estimate(cond, tol)}
