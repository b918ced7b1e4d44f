"""Effective properties and textbook bounds — oracle (TEST INFRASTRUCTURE ONLY).

Effective conductivity (motivating output P:31, Fourier law Eq 74):
    kappa_bar_ij = <kappa> delta_ij - f^(i) . theta^(j) / |Omega|
Effective stiffness (Mandel, Eq A3-A4; Eq 78-81):
    D_bar_ij = B^(i) : <C> : B^(j) - f^(i) . u^(j) / |Omega|
f^(i) is the Galerkin RHS of load i and theta^(j)/u^(j) the fluctuation solution
of load j.  Reported unsymmetrised (parity); symmetry is a test invariant.
"""
from __future__ import annotations

import numpy as np

from . import fem, greens, pcg


def effective_from_solutions(g: fem.Grid, physics: str, phase, mat, F: np.ndarray, U: np.ndarray,
                             loads=None) -> np.ndarray:
    """F, U: [nload] fields (f^(i), u^(j)) for the load vectors `loads` (default: the first
    nload unit loads).  Returns [nload][nload] = load_i.<C>.load_j - f^(i).u^(j)/|Omega|."""
    nl = F.shape[0]
    vol = g.volume()
    if loads is None:
        nv = g.d if physics == "thermal" else fem.mandel_dim(g.d)
        loads = np.eye(nv)[:nl]
    L = np.asarray(loads, dtype=float)
    if physics == "thermal":
        base = fem.phase_mean(phase, *mat) * (L @ L.T)
    else:
        (l0, m0), (l1, m1) = mat
        lam_m = fem.phase_mean(phase, l0, l1)
        mu_m = fem.phase_mean(phase, m0, m1)
        base = L @ fem.isotropic_D(g.d, lam_m, mu_m) @ L.T
    FU = np.array([[float(np.sum(F[i] * U[j])) for j in range(nl)] for i in range(nl)])
    return base - FU / vol


def centroid_flux_average(g: fem.Grid, phase, kappa, gbar, theta) -> np.ndarray:
    """<q> / (-1) = <kappa (gbar + grad theta)> with the element-mean gradient (independent
    cross-check of the f.u formula; SURVEY C4 'identity (i)')."""
    d = g.d
    G = fem.mean_shape_grad(d, g.h) / np.prod(g.h)  # element-mean gradient of each N_a
    uf = fem._pad_full(g, theta)
    grad = np.zeros((d,) + g.elem_shape)
    for ai, a in enumerate(fem.corners(d)):
        ua = fem._gather(g, uf, a)[0]
        for i in range(d):
            grad[i] += G[ai, i] * ua
    kap = fem.coeff_field(phase, *kappa)
    return np.array([np.mean(kap * (gbar[i] + grad[i])) for i in range(d)])


def voigt_reuss(v0: float, v1: float, vf1: float):
    voigt = (1 - vf1) * v0 + vf1 * v1
    reuss = 1.0 / ((1 - vf1) / v0 + vf1 / v1)
    return voigt, reuss


def hs_thermal(k0: float, k1: float, vf1: float, d: int = 3):
    """Hashin-Shtrikman bounds for an isotropic two-phase conductor in d dimensions."""
    lo_k, hi_k = (k0, k1) if k0 <= k1 else (k1, k0)
    vf_hi = vf1 if k1 >= k0 else 1 - vf1
    vf_lo = 1 - vf_hi
    lower = lo_k + vf_hi / (1.0 / (hi_k - lo_k) + vf_lo / (d * lo_k)) if hi_k > lo_k else lo_k
    upper = hi_k + vf_lo / (1.0 / (lo_k - hi_k) + vf_hi / (d * hi_k)) if hi_k > lo_k else hi_k
    return lower, upper


def laminate_elastic(d: int, normal_axis: int, D0: np.ndarray, D1: np.ndarray, vf1: float, eps_bar: np.ndarray) -> np.ndarray:
    """Textbook layer-averaging closed form: traction t and strain jump a with
    eps = eps_bar + sym(a (x) n) continuous-traction per layer.  Returns <sigma> (Mandel)."""
    import itertools
    pairs = fem._mandel_pairs(d)
    s2 = np.sqrt(2.0)

    def to_tensor(v):
        T = np.zeros((d, d))
        for m, (i, j) in enumerate(pairs):
            if i == j:
                T[i, i] = v[m]
            else:
                T[i, j] = T[j, i] = v[m] / s2
        return T

    def to_mandel(T):
        return np.array([T[i, i] if i == j else s2 * T[i, j] for (i, j) in pairs])

    n = np.zeros(d)
    n[normal_axis] = 1.0

    def acoustic(D):
        # C_nn[p,q] = n_i C_ipqj n_j computed via the Mandel operator on sym(e_q (x) n)
        M = np.zeros((d, d))
        for q in range(d):
            E = np.zeros((d, d))
            E[q] += n
            E = 0.5 * (E + E.T)
            S = to_tensor(D @ to_mandel(E))
            M[:, q] = S @ n
        return M

    eb = to_tensor(eps_bar)
    A0, A1 = acoustic(D0), acoustic(D1)
    t0 = to_tensor(D0 @ to_mandel(eb)) @ n
    t1 = to_tensor(D1 @ to_mandel(eb)) @ n
    inv0, inv1 = np.linalg.inv(A0), np.linalg.inv(A1)
    Minv = (1 - vf1) * inv0 + vf1 * inv1
    t = np.linalg.solve(Minv, (1 - vf1) * inv0 @ t0 + vf1 * inv1 @ t1)
    a0 = inv0 @ (t - t0)
    a1 = inv1 @ (t - t1)
    e0 = eb + 0.5 * (np.outer(a0, n) + np.outer(n, a0))
    e1 = eb + 0.5 * (np.outer(a1, n) + np.outer(n, a1))
    return (1 - vf1) * (D0 @ to_mandel(e0)) + vf1 * (D1 @ to_mandel(e1))


def zero_rhs_floor(g: fem.Grid, physics: str, mat, load) -> float:
    """||r0||_inf at or below this is a zero RHS up to assembly round-off (reading R7):
    1e-13 x (largest modulus) x h^(d-1) x ||load||_inf.  kappa_max (thermal) or max(lam + 2 mu)."""
    if physics == "thermal":
        mod = max(abs(mat[0]), abs(mat[1]))
    else:
        mod = max(l + 2 * m for (l, m) in mat)
    return 1e-13 * mod * float(np.prod(g.h)) / min(g.h) * float(np.max(np.abs(load)))


def solve_problem(g: fem.Grid, physics: str, phase, mat, loads, seed: int, amp: float,
                  tol: float = 1e-8, max_iter: int = 10000, fixed_iters: int = 0):
    """Full oracle pipeline for one problem: RHS (a1), G_hat (a0), Alg 2 (a2-a8), mean
    removal and effective property (a9).  Returns dict with per-load results."""
    mixed = g.bc == (0, 0, 1)
    alld = all(b == 1 for b in g.bc)
    if g.bc == (0, 1):  # 2D mixed: periodic x, Dirichlet y
        G = greens.ghat_mixed2d(g, physics, mat, seed, amp)
        applyP = lambda v: greens.apply_precond_mixed2d(G, v)  # noqa: E731
    elif alld:
        G = greens.ghat_dirichlet(g, physics, mat, seed, amp)
        applyP = lambda v: greens.apply_precond_dirichlet(G, v)  # noqa: E731
    elif mixed:
        G = greens.ghat_mixed(g, physics, mat, seed, amp)
        applyP = lambda v: greens.apply_precond_mixed(G, v)  # noqa: E731
    else:
        G = greens.ghat(g, physics, mat, seed, amp)
        applyP = lambda v: greens.apply_precond(G, v)  # noqa: E731
    F, U, its, results = [], [], [], []
    for ld in loads:
        f = fem.rhs(g, physics, phase, mat, ld)
        res = pcg.pcg(lambda v: fem.apply_K(g, physics, phase, mat, v), applyP, f, tol=tol, max_iter=max_iter,
                      fixed_iters=fixed_iters, zero_floor=zero_rhs_floor(g, physics, mat, ld))
        u = pcg.remove_mean(res.u) if all(b == 0 for b in g.bc) else res.u
        F.append(f)
        U.append(u)
        its.append(res.iterations)
        results.append(res)
    F = np.stack(F)
    U = np.stack(U)
    eff = effective_from_solutions(g, physics, phase, mat, F, U, loads)
    return {"G": G, "F": F, "U": U, "iterations": its, "results": results, "effective": eff}
