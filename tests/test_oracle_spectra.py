"""Oracle pins for the Tab 4 spectral estimate (oracle/spectra.py): the Lanczos
tridiagonal built from the Alg 1 coefficients against the eigenvalues of the assembled P A
(brute force on tiny grids), Ritz interlacing, and the FANS bounds of Tab 4's last row."""
import json
import os

import numpy as np
import pytest

from oracle import baselines, fem, greens, pcg, spectra

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _case(N, physics, kind, seed=0):
    rng = np.random.default_rng(seed)
    d = len(N)
    c = 1 if physics == "thermal" else d
    g = fem.Grid(N, c=c, h=1.0 / N[0])
    ph = (rng.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 10.0) if physics == "thermal" else ((0.6, 0.4), (6.0, 3.5))
    A = fem.assemble_dense(g, physics, ph, mat)
    if kind == "identity":
        P, aP = np.eye(A.shape[0]), (lambda r: r.copy())
    elif kind == "jacobi":
        dg = baselines.diag_K(g, physics, ph, mat)
        P, aP = np.diag(1.0 / dg.reshape(-1)), (lambda r: r / dg)
    else:
        G = greens.ghat(g, physics, mat, 7, 0.1 if physics == "thermal" else 0.05)
        P, aP = greens.dense_P(G, N), (lambda r: greens.apply_precond(G, r))
    aA = lambda v: fem.apply_K(g, physics, ph, mat, v)  # noqa: E731
    f = aA(rng.standard_normal(g.field_shape()))  # in range(A): consistent periodic system
    return g, A, P, aA, aP, f, c


@pytest.mark.parametrize("N,physics,kind", [((6, 6), "thermal", "identity"), ((6, 6), "thermal", "jacobi"),
                                            ((6, 6), "thermal", "uno"), ((4, 4, 4), "thermal", "uno"),
                                            ((4, 4), "elastic", "uno"), ((4, 4), "elastic", "jacobi")])
def test_ritz_extremes_match_dense_spectrum(N, physics, kind):
    # run Alg 1 to (near) termination: the extreme Ritz values equal the extreme eigenvalues of
    # P A on the range (brute force: np.linalg.eigvals of the assembled product)
    g, A, P, aA, aP, f, c = _case(N, physics, kind)
    res = pcg.pcg(aA, aP, f, tol=1e-13, max_iter=6 * A.shape[0])
    assert res.converged
    lo, hi = spectra.ritz_extremes(res.gamma, res.alpha)
    ev = spectra.dense_spectrum(A, P, c)
    # the largest Ritz value converges first (1e-8); the smallest one approaches lambda_min from
    # above and converges last onto near-degenerate pairs (1e-4) — a wrong coefficient in T moves
    # the extremes by O(1) or outside the spectrum
    assert abs(hi - ev[-1]) <= 1e-8 * ev[-1], (hi, ev[-1])
    assert ev[0] - 1e-10 * ev[-1] <= lo <= ev[0] * (1 + 1e-4), (lo, ev[0])


@pytest.mark.parametrize("m", [2, 4, 7])
def test_ritz_values_interlace(m):
    # after m < n steps the Ritz values lie inside [lambda_min, lambda_max] of P A and the
    # extreme ones move outwards with m (Cauchy interlacing of the Lanczos tridiagonals)
    g, A, P, aA, aP, f, c = _case((6, 6), "thermal", "uno", seed=3)
    ev = spectra.dense_spectrum(A, P, c)
    r_m = pcg.pcg(aA, aP, f, fixed_iters=m)
    r_m1 = pcg.pcg(aA, aP, f, fixed_iters=m + 1)
    lo, hi = spectra.ritz_extremes(r_m.gamma, r_m.alpha)
    lo1, hi1 = spectra.ritz_extremes(r_m1.gamma, r_m1.alpha)
    tol = 1e-10 * ev[-1]
    assert ev[0] - tol <= lo1 <= lo + tol and hi - tol <= hi1 <= ev[-1] + tol


def test_single_step_tridiagonal_is_rayleigh_quotient():
    # m = 1: T = [1/alpha_0] = (s.A s)/(r.s) with s = P r, the Rayleigh quotient of P A at s in the
    # P^-1 inner product (<s, P A s> / <s, s> with <x, y> = x.P^-1 y) — written out from the
    # definitions, not from lanczos_T
    g, A, P, aA, aP, f, c = _case((6, 6), "thermal", "jacobi", seed=5)
    s = aP(f)
    rq = float(np.sum(s * aA(s)) / np.sum(f * s))
    res = pcg.pcg(aA, aP, f, fixed_iters=1)
    assert abs(spectra.lanczos_T(res.gamma, res.alpha)[0, 0] - rq) <= 1e-13 * rq


def test_fans_ritz_values_inside_table4_bounds():
    # Tab 4 FANS row: every eigenvalue of P_FANS A lies in [kappa_min, kappa_max]/kappa_r
    # = [1/3, 5/3] for kappa 1/0.2, so every Ritz value does too, and the converged extremes
    # approach the bounds for a two-phase 16^2 microstructure
    tab = json.load(open(os.path.join(GOLD, "table4.json")))
    mat = (tab["fans_material"]["kappa0"], tab["fans_material"]["kappa1"])
    N = (16, 16)
    g = fem.Grid(N)
    ph = (np.random.default_rng(1).random(g.elem_shape) < 0.5).astype(np.uint8)
    G = greens.ghat(g, "thermal", mat, 0, 0.0)
    aA = lambda v: fem.apply_K(g, "thermal", ph, mat, v)  # noqa: E731
    f = fem.rhs(g, "thermal", ph, mat, np.array([1.0, 0.0]))
    res = pcg.pcg(aA, lambda r: greens.apply_precond(G, r), f, tol=1e-12, max_iter=500)
    T = spectra.lanczos_T(res.gamma, res.alpha)
    ev = np.linalg.eigvalsh(T)
    assert ev[0] >= 1 / 3 - 1e-10 and ev[-1] <= 5 / 3 + 1e-10
    row = spectra.table4_row(ev[0], ev[-1], tab["tol"])
    assert row["cond"] <= 5.0 + 1e-9 and row["C_CG"] <= pcg.cg_rate(5.0) + 1e-12
