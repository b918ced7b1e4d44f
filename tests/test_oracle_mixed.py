"""Pins for the mixed-BC oracle (periodic x, y; Dirichlet z; U = F_x (x) F_y (x) DST-I_z —
Table 1 row "Mixed").  Not gpu."""
import numpy as np
import pytest

from oracle import fem, greens, homog, pcg, transform

RNG = np.random.default_rng(2024)


@pytest.mark.parametrize("nm1", [3, 7, 15])
def test_dst1_matrix_orthonormal_and_sine_eigenvector(nm1):
    S = transform.dst1_matrix(nm1)
    assert np.max(np.abs(S @ S - np.eye(nm1))) < 1e-13     # symmetric, self-inverse
    assert np.max(np.abs(S - S.T)) < 1e-14
    N = nm1 + 1
    j = np.arange(1, N)
    for m in (1, nm1):                                     # SPEC S:216 sine-basis example
        x = np.sin(np.pi * m * j / N)
        y = S @ x
        e = np.zeros(nm1)
        e[m - 1] = 1.0
        assert np.max(np.abs(y - np.linalg.norm(x) * e)) < 1e-12
    # the 1D Dirichlet 3-point Laplacian is diagonalised exactly
    L = 2 * np.eye(nm1) - np.eye(nm1, k=1) - np.eye(nm1, k=-1)
    D = S @ L @ S
    assert np.max(np.abs(D - np.diag(np.diag(D)))) < 1e-12
    assert np.max(np.abs(np.diag(D) - (2 - 2 * np.cos(np.pi * j / N)))) < 1e-12


def test_forward_mixed_matches_dense():
    shape = (5, 4, 6)
    x = RNG.standard_normal(shape)
    T = transform.dense_T_mixed(shape)
    full = (T @ x.reshape(-1)).reshape(shape)
    xh = transform.forward_mixed(x[None])[0]
    assert np.max(np.abs(xh - full[..., :4])) < 1e-13
    assert np.max(np.abs(transform.inverse_mixed(transform.forward_mixed(x[None]), shape)[0] - x)) < 1e-13


def test_thermal_mixed_exact_inverse():
    # homogeneous medium, seed 0: F(x)F(x)DST-I diagonalises K_r exactly -> P K u = u
    g = fem.Grid((6, 4, 8), bc=(0, 0, 1), h=1 / 8)
    ph = np.zeros(g.elem_shape, np.uint8)
    mat = (2.0, 2.0)
    G = greens.ghat_mixed(g, "thermal", mat, 0, 0.0)
    u = RNG.standard_normal(g.field_shape())
    assert np.max(np.abs(greens.apply_precond_mixed(G, fem.apply_K(g, "thermal", ph, mat, u)) - u)) < 1e-12


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_mixed_symbol_is_diagonal_block_of_dense(physics):
    c = 1 if physics == "thermal" else 3
    g = fem.Grid((4, 6, 6), bc=(0, 0, 1), c=c, h=1 / 6)
    ph = np.zeros(g.elem_shape, np.uint8)
    ref = 1.3 if physics == "thermal" else (0.8, 0.6)
    mat = (ref, ref)
    A = fem.assemble_dense(g, physics, ph, mat)
    T = np.kron(np.eye(c), transform.dense_T_mixed(g.node_shape))
    D = T @ A @ T.conj().T
    n = g.n
    blk = np.array([[np.diag(D[a * n:(a + 1) * n, b * n:(b + 1) * n]) for b in range(c)] for a in range(c)])
    probe = greens.symbol_probe_mixed(g, physics, ref).reshape(c, c, -1)
    assert np.max(np.abs(blk.imag)) < 1e-12
    assert np.max(np.abs(blk.real - probe)) < 1e-12 * np.abs(probe).max()


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_mixed_perturbed_symbol_and_lemma1(physics):
    c = 1 if physics == "thermal" else 3
    g = fem.Grid((4, 4, 4), bc=(0, 0, 1), c=c, h=1 / 4)
    mat = (1.0, 10.0) if physics == "thermal" else ((0.58, 0.38), (2.78, 4.17))
    G = greens.ghat_mixed(g, physics, mat, 31, 0.1 if c == 1 else 0.05)
    # multiplier symmetric under (kx, ky) -> (-kx, -ky) at fixed sine mode (Eq 16 on Fourier axes)
    Gm = np.roll(np.flip(np.roll(np.flip(G, axis=-1), 1, axis=-1), axis=-2), 1, axis=-2)
    assert np.array_equal(G, Gm)
    ok, lo, hi = greens.eq55_check(np.concatenate([np.zeros((c, c, 1)), G.reshape(c, c, -1)], axis=-1))
    assert ok and lo > 0
    P = greens.dense_P_mixed(G, g.node_shape)                 # Lemma 1 with the mixed transform
    ev = np.sort(np.linalg.eigvalsh(P))
    evb = np.sort(np.linalg.eigvalsh(np.moveaxis(G.reshape(c, c, -1), -1, 0)).reshape(-1))
    assert np.max(np.abs(ev - evb)) < 1e-9 * evb.max()


@pytest.mark.parametrize("physics,N", [("thermal", (8, 4, 8)), ("elastic", (4, 4, 6))])
def test_mixed_pcg_vs_dense_solve(physics, N):
    c = 1 if physics == "thermal" else 3
    g = fem.Grid(N, bc=(0, 0, 1), c=c, h=1 / N[0])
    ph = (RNG.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 20.0) if physics == "thermal" else ((0.58, 0.38), (2.78, 4.17))
    load = np.eye(3 if c == 1 else 6)[0]
    out = homog.solve_problem(g, physics, ph, mat, [load], 7, 0.1 if c == 1 else 0.05, tol=1e-12)
    A = fem.assemble_dense(g, physics, ph, mat)
    f = fem.rhs(g, physics, ph, mat, load)
    x = np.linalg.solve(A, f.reshape(-1)).reshape(f.shape)   # Dirichlet: SPD, unique
    assert out["results"][0].converged
    assert np.linalg.norm(out["U"][0] - x) <= 1e-9 * np.linalg.norm(x)
