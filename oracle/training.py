"""Second-order UNO preconditioner training, §4.4 Alg 4 and App. B
 — oracle (TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference arm use oracle/).  Periodic grids, T = orthonormal DFT.

Training pairs (Eq 58, 60): r^(j) = f^(j), s^(j) = A^{-1} f^(j) = u^(j).
Features (Eq 62, 67, B.2) on the full frequency grid, component a = 0..c-1:
    alpha_ab(k) = (1/Ns) sum_j Re(conj(r^_a) r^_b)      (alpha_1 = alpha_xx, alpha_3 = 2 alpha_xy, ...)
    beta_ab(k)  = (2/Ns) sum_j Re(conj(r^_a) s^_b)
so that per frequency the loss (Eq 63) is
    l(k) = sum_ab (Q^2)_ab A_ab - sum_ab Q_ab B_ab + delta,   A_ab = Re(conj r^_a r^_b) averaged,
i.e. L(v) = 1/2 v^T H(alpha) v - beta . v + delta with H the Hessian of Eq 66 / 71 / B.2 and v the
unique entries of Q(k) in Eq B7 order (v1=Q11, v2=Q22, v3=Q12, v4=Q33, v5=Q23, v6=Q13).
Parametrization (Eq 43-45, B5): v(k) = psi(theta_0) + [k in K] psi(theta_{p(k)}), psi(t) = t^2 (c=1),
psi = L L^T from the C weights (c=2, 3); K = {k : |k_i| <= M on every axis} (Table 1 "Periodic"),
conjugate modes {k, -k} share one weight vector (K_c, Eq 43).  Newton-Raphson (Alg 4 l.4-7) on
theta with the exact gradient / Hessian of Eq 72; the Hessian couples theta_0 with every mode
block, so the step is solved by a Schur complement on theta_0 (the band structure of Alg 4 l.6).
"""
from __future__ import annotations

import numpy as np

from . import greens

# unique entries (Eq B7 order) -> (a, b) component pairs
PAIRS = {1: [(0, 0)], 2: [(0, 0), (1, 1), (0, 1)], 3: [(0, 0), (1, 1), (0, 1), (2, 2), (1, 2), (0, 2)]}


def unpack(v: np.ndarray, c: int) -> np.ndarray:
    """(C, ...) unique entries -> (c, c, ...) symmetric Q."""
    Q = np.zeros((c, c) + v.shape[1:])
    for m, (a, b) in enumerate(PAIRS[c]):
        Q[a, b] = v[m]
        Q[b, a] = v[m]
    return Q


def fft_full(x: np.ndarray) -> np.ndarray:
    """Orthonormal DFT over the spatial axes of a (c, ...) field (T of Eq 47)."""
    return np.fft.fftn(x, axes=tuple(range(1, x.ndim)), norm="ortho")


def features(R: list, S: list):
    """A[a][b](k) = (1/Ns) sum_j Re(conj r^_a r^_b);  B[a][b](k) = (1/Ns) sum_j Re(conj r^_a s^_b);
    delta = (1/Ns) sum_j ||s_j||^2 (Eq 62-67, B.2).  R, S: lists of (c, ...) fields."""
    ns = len(R)
    c = R[0].shape[0]
    A = np.zeros((c, c) + R[0].shape[1:])
    B = np.zeros((c, c) + R[0].shape[1:])
    delta = 0.0
    for r, s in zip(R, S):
        rh, sh = fft_full(r), fft_full(s)
        for a in range(c):
            for b in range(c):
                A[a, b] += np.real(np.conj(rh[a]) * rh[b]) / ns
                B[a, b] += np.real(np.conj(rh[a]) * sh[b]) / ns
        delta += float(np.sum(s * s)) / ns
    return A, B, delta


def paper_features(A: np.ndarray, B: np.ndarray):
    """alpha_m, beta_m of Eq 67 / (c=2) / B.2 from A, B: alpha for the Q^2 terms, beta = 2 sym B."""
    c = A.shape[0]
    al, be = [], []
    for a, b in PAIRS[c]:
        al.append(A[a, a] if a == b else A[a, b] + A[b, a])
        be.append(2 * B[a, a] if a == b else 2 * (B[a, b] + B[b, a]))
    return np.stack(al), np.stack(be)


def loss_direct(v: np.ndarray, R: list, S: list) -> float:
    """(1/Ns) sum_j || T^H Q T r_j - s_j ||^2 (Eq 59) by applying the preconditioner."""
    c = R[0].shape[0]
    Q = unpack(v, c)
    tot = 0.0
    for r, s in zip(R, S):
        rh = fft_full(r)
        sh = np.einsum("ab...,b...->a...", Q, rh)
        pr = np.fft.ifftn(sh, axes=tuple(range(1, r.ndim)), norm="ortho").real
        tot += float(np.sum((pr - s) ** 2))
    return tot / len(R)


def loss_features(v: np.ndarray, A: np.ndarray, B: np.ndarray, delta: float) -> float:
    """Eq 63 summed over k: sum_k [ sum_ab (Q^2)_ab A_ab - 2 sum_ab Q_ab B_ab ] + delta."""
    c = A.shape[0]
    Q = unpack(v, c)
    Q2 = np.einsum("ab...,bc...->ac...", Q, Q)
    return float(np.sum(Q2 * A) - 2.0 * np.sum(Q * B) + delta)


def hess_v(A: np.ndarray) -> np.ndarray:
    """d^2 l / dv dv per frequency (C, C, ...) — Eq 66 (c=1), Eq 71 (c=2), B.2 (c=3): the loss is
    quadratic in v, l = 1/2 v^T H v - beta . v + delta, H_mn = d^2 sum_ab (Q^2)_ab A_ab / dv_m dv_n."""
    c = A.shape[0]
    C = len(PAIRS[c])
    H = np.zeros((C, C) + A.shape[2:])
    E = []
    for m in range(C):
        e = np.zeros((C,) + A.shape[2:])
        e[m] = 1.0
        E.append(unpack(e, c))
    for m in range(C):
        for n in range(C):
            # d^2/dv_m dv_n of tr(Q Q A) = tr((E_m E_n + E_n E_m) A)
            M = np.einsum("ab...,bc...->ac...", E[m], E[n]) + np.einsum("ab...,bc...->ac...", E[n], E[m])
            H[m, n] = np.sum(M * A, axis=(0, 1))
    return H


def psi(theta: np.ndarray, c: int) -> np.ndarray:
    """Local parametrization psi: R^C -> Sym+ (Eq 45 / B5), returned as unique entries (C, ...)."""
    t = theta
    if c == 1:
        return t[0:1] ** 2
    if c == 2:
        return np.stack([t[0] ** 2, t[1] ** 2 + t[2] ** 2, t[0] * t[2]])
    t1, t2, t3, t4, t5, t6 = t
    return np.stack([t1 * t1, t2 * t2 + t3 * t3, t1 * t3, t4 * t4 + t5 * t5 + t6 * t6, t2 * t5 + t3 * t6, t1 * t6])


def psi_jac(theta: np.ndarray, c: int, eps: float = 0.0):
    """dpsi/dtheta (C, C, ...) and d2psi/dtheta2 (C, C, C) (constant: psi is quadratic)."""
    C = theta.shape[0]
    J = np.zeros((C, C) + theta.shape[1:])
    D2 = np.zeros((C, C, C))
    for m in range(C):  # second derivatives from psi at unit vectors: psi is a quadratic form per entry
        for i in range(C):
            for k in range(C):
                ei = np.zeros(C)
                ek = np.zeros(C)
                ei[i] = 1.0
                ek[k] = 1.0
                D2[m, i, k] = psi(ei + ek, c)[m] - psi(ei, c)[m] - psi(ek, c)[m]
                if i == k:
                    D2[m, i, k] = 2.0 * psi(ei, c)[m]
    for m in range(C):
        J[m] = np.einsum("ik,k...->i...", D2[m], theta)
    return J, D2


def mode_pairs(shape, M: int):
    """p(k): index of the conjugate pair {k, -k} of every k in K = {|k_i| <= M} (signed), else -1."""
    grids = np.meshgrid(*[np.fft.fftfreq(n, 1.0 / n).astype(int) for n in shape], indexing="ij")
    inK = np.ones(shape, dtype=bool)
    for gk in grids:
        inK &= np.abs(gk) <= M
    can = greens.canon_index(shape)
    ids = np.full(shape, -1, dtype=np.int64)
    uniq = np.unique(can[inK])
    lut = {int(u): i for i, u in enumerate(uniq)}
    for idx in zip(*np.nonzero(inK)):
        ids[idx] = lut[int(can[idx])]
    return ids, len(uniq)


def symbol(theta0: np.ndarray, thetas: np.ndarray, ids: np.ndarray, c: int) -> np.ndarray:
    v = np.broadcast_to(psi(theta0[:, None], c)[:, 0].reshape((-1,) + (1,) * ids.ndim), (len(PAIRS[c]),) + ids.shape).copy()
    sel = ids >= 0
    v[:, sel] += psi(thetas[:, ids[sel]], c)
    return v


def newton(A, B, delta, M: int, theta0, thetas, epochs: int = 10, ids=None, npair=None, max_halvings: int = 30):
    """Alg 4: Newton-Raphson on (theta_0, theta_p).  Returns theta0, thetas, loss history.
    Reading (R15): the loss is quartic in theta, so far from the optimum a full Newton
    step can increase it; the step is then halved until the loss does not increase (backtracking;
    after max_halvings without decrease theta is kept), which leaves the quadratically convergent
    full steps near the optimum untouched."""
    c = A.shape[0]
    C = len(PAIRS[c])
    shape = A.shape[2:]
    if ids is None:
        ids, npair = mode_pairs(shape, M)
    al, be = paper_features(A, B)
    Hv = hess_v(A)  # (C, C, ...)
    hist = []
    for _ in range(epochs):
        v = symbol(theta0, thetas, ids, c)
        hist.append(loss_features(v, A, B, delta))
        gv = np.einsum("mn...,n...->m...", Hv, v) - be  # dl/dv per k (Eq 66 / 71 / B.2)
        J0, D2 = psi_jac(theta0[:, None], c)
        J0 = J0[..., 0]
        # theta_0 block (sums over all k)
        gvf = gv.reshape(C, -1)
        Hvf = Hv.reshape(C, C, -1)
        g0 = np.einsum("mi,mk->i", J0, gvf)
        H00 = np.einsum("mi,mnk,nj->ij", J0, Hvf, J0) + np.einsum("mk,mij->ij", gvf, D2)
        # mode blocks: sums over the members of each conjugate pair
        sel = ids >= 0
        P = npair
        gvs = gv[:, sel]
        Hvs = Hv[:, :, sel]
        pid = ids[sel]
        Jp, _ = psi_jac(thetas, c)  # (C, C, P)
        Jk = Jp[:, :, pid]
        gp = np.zeros((C, P))
        np.add.at(gp.T, pid, np.einsum("mik,mk->ki", Jk, gvs))
        Hpp = np.zeros((P, C, C))
        np.add.at(Hpp, pid, np.einsum("mik,mnk,njk->kij", Jk, Hvs, Jk) + np.einsum("mk,mij->kij", gvs, D2))
        H0p = np.zeros((P, C, C))
        np.add.at(H0p, pid, np.einsum("mi,mnk,njk->kij", J0, Hvs, Jk))
        # Schur complement on theta_0
        Hinv = np.linalg.inv(Hpp)
        S = H00 - np.einsum("pij,pjk,plk->il", H0p, Hinv, H0p)
        rhs = g0 - np.einsum("pij,pjk,kp->i", H0p, Hinv, gp)
        d0 = np.linalg.solve(S, rhs)
        dp = np.einsum("pij,jp->ip", Hinv, gp - np.einsum("pji,j->ip", H0p, d0))
        t = 1.0
        for _ in range(max_halvings):
            cand0, cands = theta0 - t * d0, thetas - t * dp
            if loss_features(symbol(cand0, cands, ids, c), A, B, delta) <= hist[-1]:
                theta0, thetas = cand0, cands
                break
            t *= 0.5  # no decrease after max_halvings: stationary to round-off, keep theta
    v = symbol(theta0, thetas, ids, c)
    hist.append(loss_features(v, A, B, delta))
    return theta0, thetas, hist
