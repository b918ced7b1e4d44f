"""Pins for the all-Dirichlet oracle (U = DST-I on every axis; Table 1 row "Dirichlet", P:451;
SURVEY §8(f) rank 1).  Not gpu."""
import numpy as np
import pytest

from oracle import fem, greens, homog, transform

RNG = np.random.default_rng(4242)


def test_dense_transform_orthonormal_and_matches_fast():
    shape = (3, 4, 5)
    T = transform.dense_T_dirichlet(shape)
    assert np.max(np.abs(T @ T.T - np.eye(T.shape[0]))) < 1e-13
    x = RNG.standard_normal((1,) + shape)
    assert np.max(np.abs(transform.forward_dirichlet(x)[0].reshape(-1) - T @ x.reshape(-1))) < 1e-13
    assert np.max(np.abs(transform.inverse_dirichlet(transform.forward_dirichlet(x)) - x)) < 1e-13


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_symbol_is_diagonal_block_of_dense(physics):
    c = 1 if physics == "thermal" else 3
    g = fem.Grid((4, 5, 4), bc=(1, 1, 1), c=c, h=1 / 4)
    ref = 1.7 if physics == "thermal" else (0.8, 0.6)
    A = fem.assemble_dense(g, physics, np.zeros(g.elem_shape, np.uint8), (ref, ref))
    T = np.kron(np.eye(c), transform.dense_T_dirichlet(g.node_shape))
    D = T @ A @ T.T
    n = g.n
    blk = np.array([[np.diag(D[a * n:(a + 1) * n, b * n:(b + 1) * n]) for b in range(c)] for a in range(c)])
    probe = greens.symbol_probe_dirichlet(g, physics, ref).reshape(c, c, -1)
    assert np.max(np.abs(blk - probe)) < 1e-12 * np.abs(probe).max()
    if physics == "thermal":  # the sine basis diagonalises the reference operator exactly
        assert np.max(np.abs(D - np.diag(np.diag(D)))) < 1e-12 * np.abs(D).max()
    else:  # elastic: the diagonal block itself is diagonal (couplings odd in two offsets drop)
        off = blk.copy()
        for a in range(3):
            off[a, a] = 0
        assert np.max(np.abs(off)) < 1e-12 * np.abs(probe).max()


def test_thermal_exact_inverse():
    g = fem.Grid((5, 4, 6), bc=(1, 1, 1), h=1 / 5)
    ph = np.zeros(g.elem_shape, np.uint8)
    G = greens.ghat_dirichlet(g, "thermal", (2.5, 2.5), 0, 0.0)
    u = RNG.standard_normal(g.field_shape())
    PKu = greens.apply_precond_dirichlet(G, fem.apply_K(g, "thermal", ph, (2.5, 2.5), u))
    assert np.max(np.abs(PKu - u)) < 1e-12


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_perturbed_symbol_lemma1_and_eq55(physics):
    c = 1 if physics == "thermal" else 3
    g = fem.Grid((4, 4, 4), bc=(1, 1, 1), c=c, h=1 / 4)
    mat = (1.0, 10.0) if physics == "thermal" else ((0.58, 0.38), (2.78, 4.17))
    G = greens.ghat_dirichlet(g, physics, mat, 55, 0.1 if c == 1 else 0.05)
    ok, lo, _ = greens.eq55_check(np.concatenate([np.zeros((c, c, 1)), G.reshape(c, c, -1)], axis=-1))
    assert ok and lo > 0
    P = greens.dense_P_dirichlet(G, g.node_shape)
    ev = np.sort(np.linalg.eigvalsh(P))
    evb = np.sort(np.linalg.eigvalsh(np.moveaxis(G.reshape(c, c, -1), -1, 0)).reshape(-1))
    assert np.max(np.abs(ev - evb)) < 1e-9 * evb.max()


@pytest.mark.parametrize("physics,N", [("thermal", (6, 5, 7)), ("elastic", (4, 5, 4))])
def test_pcg_vs_dense_solve(physics, N):
    c = 1 if physics == "thermal" else 3
    g = fem.Grid(N, bc=(1, 1, 1), c=c, h=1 / N[0])
    ph = (RNG.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 20.0) if physics == "thermal" else ((0.58, 0.38), (2.78, 4.17))
    load = np.eye(3 if c == 1 else 6)[1]
    out = homog.solve_problem(g, physics, ph, mat, [load], 5, 0.1 if c == 1 else 0.05, tol=1e-12)
    A = fem.assemble_dense(g, physics, ph, mat)
    f = fem.rhs(g, physics, ph, mat, load)
    x = np.linalg.solve(A, f.reshape(-1)).reshape(f.shape)
    assert out["results"][0].converged
    assert np.linalg.norm(out["U"][0] - x) <= 1e-9 * np.linalg.norm(x)
