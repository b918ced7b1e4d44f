"""Pins for oracle/training.py (second-order UNO training, Alg 4, Eq 59-72, App. B; P:543-667,
1010-1036).  Not gpu."""
import numpy as np
import pytest

from oracle import fem, greens, pcg, training

RNG = np.random.default_rng(99)


def _pairs(c, shape, ns):
    R = [RNG.standard_normal((c,) + shape) for _ in range(ns)]
    S = [RNG.standard_normal((c,) + shape) for _ in range(ns)]
    return R, S


@pytest.mark.parametrize("c", [1, 2, 3])
def test_feature_loss_equals_direct_loss(c):
    # Eq 63-67 / B.2 (features) == Eq 59 (apply T^H Q T to every sample) for any symmetric Q(k)
    shape = (4, 6) if c == 2 else (4, 5, 6)
    R, S = _pairs(c, shape, 3)
    A, B, delta = training.features(R, S)
    C = len(training.PAIRS[c])
    v = RNG.standard_normal((C,) + shape)
    # a symbol must be conjugate-symmetric for T^H Q T to be real: symmetrise over k -> -k
    v = 0.5 * (v + np.roll(np.flip(v, axis=tuple(range(1, v.ndim))), 1, axis=tuple(range(1, v.ndim))))
    assert abs(training.loss_features(v, A, B, delta) - training.loss_direct(v, R, S)) < 1e-10 * training.loss_direct(v, R, S)


@pytest.mark.parametrize("c", [1, 3])
def test_quadratic_form_hessian_and_gradient(c):
    shape = (3, 4, 5)
    R, S = _pairs(c, shape, 2)
    A, B, delta = training.features(R, S)
    al, be = training.paper_features(A, B)
    H = training.hess_v(A)
    C = H.shape[0]
    for _ in range(3):
        v = RNG.standard_normal((C,) + shape)
        q = 0.5 * np.sum(np.einsum("m...,mn...,n...->...", v, H, v)) - np.sum(be * v) + delta
        assert abs(q - training.loss_features(v, A, B, delta)) < 1e-10 * abs(q)
    if c == 3:  # B.2's printed Hessian: H[0,0] = 2 alpha_1, H[0,2] = alpha_3, H[2,2] = 2(alpha_1 + alpha_2)
        assert np.allclose(H[0, 0], 2 * al[0]) and np.allclose(H[0, 2], al[2])
        assert np.allclose(H[2, 2], 2 * (al[0] + al[1])) and np.allclose(H[4, 4], 2 * (al[1] + al[3]))
    else:  # Eq 66: 2 diag(alpha_1)
        assert np.allclose(H[0, 0], 2 * al[0])


@pytest.mark.parametrize("c", [1, 3])
def test_psi_derivatives(c):
    C = len(training.PAIRS[c])
    th = RNG.standard_normal((C, 4))
    J, D2 = training.psi_jac(th, c)
    e = 1e-6
    for i in range(C):
        dt = np.zeros_like(th)
        dt[i] = e
        fd = (training.psi(th + dt, c) - training.psi(th - dt, c)) / (2 * e)
        assert np.max(np.abs(fd - J[:, i])) < 1e-8
    # psi is SPD-valued (Cholesky-like, Eq 45 / B5)
    Q = training.unpack(training.psi(th, c), c)
    for k in range(4):
        assert np.linalg.eigvalsh(Q[..., k]).min() >= -1e-14


def _solver_pairs(n_samples, N=8):
    """Training pairs of Eq 60 from our own oracle solves: r = f, s = u (mean-free)."""
    g = fem.Grid((N, N, N), h=1 / N)
    R, S = [], []
    for j in range(n_samples):
        ph = (np.random.default_rng(500 + j).random(g.elem_shape) < 0.3).astype(np.uint8)
        mat = (1.0, 5.0 + 5 * j)
        f = fem.rhs(g, "thermal", ph, mat, np.eye(3)[j % 3])
        G = greens.ghat(g, "thermal", mat, 0, 0.0)
        u = pcg.remove_mean(pcg.pcg(lambda v: fem.apply_K(g, "thermal", ph, mat, v), lambda v: greens.apply_precond(G, v),
                                    f, tol=1e-12).u)
        R.append(f)
        S.append(u)
    return g, R, S


def test_newton_decreases_loss_to_stationary_point():
    g, R, S = _solver_pairs(4)
    A, B, delta = training.features(R, S)
    shape = A.shape[2:]
    M = 2
    ids, npair = training.mode_pairs(shape, M)
    # initial guess: FANS symbol of the mean contrast split into bypass + modes
    G = greens.ghat(g, "thermal", (1.0, 12.5), 0, 0.0)[0, 0]
    gm = float(np.median(G[G > 0]))
    theta0 = np.array([np.sqrt(gm)])
    thetas = np.zeros((1, npair))
    for idx in zip(*np.nonzero(ids >= 0)):
        thetas[0, ids[idx]] = np.sqrt(max(G[idx] - gm, 0.0) + 1e-3 * gm)
    t0, ts, hist = training.newton(A, B, delta, M, theta0, thetas, epochs=12)
    assert hist[-1] < hist[0]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist, hist[1:]))  # monotone (backtracking)
    # stationary: the gradient of L w.r.t. v vanishes on the trained modes' span
    assert (hist[-2] - hist[-1]) <= 1e-9 * abs(hist[-1])


def test_trained_preconditioner_is_spd_and_converges():
    # the trained symbol is SPD by construction (psi, Lemma 1) -> PCG converges on a held-out problem
    g, R, S = _solver_pairs(4)
    A, B, delta = training.features(R, S)
    shape = A.shape[2:]
    ids, npair = training.mode_pairs(shape, 2)
    G = greens.ghat(g, "thermal", (1.0, 12.5), 0, 0.0)[0, 0]
    gm = float(np.median(G[G > 0]))
    thetas = np.zeros((1, npair))
    for idx in zip(*np.nonzero(ids >= 0)):
        thetas[0, ids[idx]] = np.sqrt(max(G[idx] - gm, 0.0) + 1e-3 * gm)
    t0, ts, _ = training.newton(A, B, delta, 2, np.array([np.sqrt(gm)]), thetas, epochs=10)
    v = training.symbol(t0, ts, ids, 1)
    assert v.min() > 0
    Gl = v.reshape((1, 1) + shape).copy()
    Gl[..., 0, 0, 0] = 0.0  # shares the periodic null space
    ph = (np.random.default_rng(999).random(g.elem_shape) < 0.3).astype(np.uint8)
    f = fem.rhs(g, "thermal", ph, (1.0, 20.0), np.eye(3)[0])
    res = pcg.pcg(lambda x: fem.apply_K(g, "thermal", ph, (1.0, 20.0), x), lambda x: greens.apply_precond(Gl, x), f,
                  tol=1e-8)
    assert res.converged and res.iterations < 80
