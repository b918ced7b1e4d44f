"""Pins for the 2D non-periodic oracles: Dirichlet (DST-I on both axes, Table 1 row "Dirichlet",
P:451) and mixed (F_x (x) S_y, Table 1 row "Mixed") for thermal and plane elasticity
(§6 2D studies P:815-853).  Not gpu."""
import numpy as np
import pytest

from oracle import fem, greens, homog, transform

RNG = np.random.default_rng(8080)


def test_mixed2d_transform():
    shape = (5, 6)
    T = transform.dense_T_mixed2d(shape)
    assert np.max(np.abs(T @ T.conj().T - np.eye(T.shape[0]))) < 1e-13
    x = RNG.standard_normal((1,) + shape)
    full = (T @ x.reshape(-1)).reshape(shape)
    assert np.max(np.abs(transform.forward_mixed2d(x)[0] - full[:, :4])) < 1e-13
    assert np.max(np.abs(transform.inverse_mixed2d(transform.forward_mixed2d(x), shape) - x)) < 1e-13


@pytest.mark.parametrize("bc", [(1, 1), (0, 1)])
@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_symbol_is_diagonal_block_of_dense(bc, physics):
    c = 1 if physics == "thermal" else 2
    g = fem.Grid((6, 6), bc=bc, c=c)
    ref = 1.4 if physics == "thermal" else (0.7, 0.9)
    A = fem.assemble_dense(g, physics, np.zeros(g.elem_shape, np.uint8), (ref, ref))
    if bc == (1, 1):
        T = np.kron(np.eye(c), transform.dense_T_dirichlet(g.node_shape))
        probe = greens.symbol_probe_dirichlet(g, physics, ref)
    else:
        T = np.kron(np.eye(c), transform.dense_T_mixed2d(g.node_shape))
        probe = greens.symbol_probe_mixed2d(g, physics, ref)
    D = T @ A @ T.conj().T
    n = g.n
    blk = np.array([[np.diag(D[a * n:(a + 1) * n, b * n:(b + 1) * n]) for b in range(c)] for a in range(c)])
    assert np.max(np.abs(blk.imag)) < 1e-12
    assert np.max(np.abs(blk.real - probe.reshape(c, c, -1))) < 1e-12 * np.abs(probe).max()
    if physics == "thermal":  # exact diagonalisation
        assert np.max(np.abs(D - np.diag(np.diag(D)))) < 1e-12 * np.abs(D).max()


@pytest.mark.parametrize("bc", [(1, 1), (0, 1)])
def test_thermal_exact_inverse(bc):
    g = fem.Grid((8, 6), bc=bc)
    ph = np.zeros(g.elem_shape, np.uint8)
    u = RNG.standard_normal(g.field_shape())
    Ku = fem.apply_K(g, "thermal", ph, (3.0, 3.0), u)
    if bc == (1, 1):
        z = greens.apply_precond_dirichlet(greens.ghat_dirichlet(g, "thermal", (3.0, 3.0), 0, 0.0), Ku)
    else:
        z = greens.apply_precond_mixed2d(greens.ghat_mixed2d(g, "thermal", (3.0, 3.0), 0, 0.0), Ku)
    assert np.max(np.abs(z - u)) < 1e-12


@pytest.mark.parametrize("bc", [(1, 1), (0, 1)])
@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_perturbed_lemma1_eq55(bc, physics):
    c = 1 if physics == "thermal" else 2
    g = fem.Grid((6, 6), bc=bc, c=c)
    mat = (1.0, 10.0) if c == 1 else ((0.58, 0.38), (2.78, 4.17))
    if bc == (1, 1):
        G = greens.ghat_dirichlet(g, physics, mat, 17, 0.1 if c == 1 else 0.05)
        P = greens.dense_P_dirichlet(G, g.node_shape)
    else:
        G = greens.ghat_mixed2d(g, physics, mat, 17, 0.1 if c == 1 else 0.05)
        Gm = np.roll(np.flip(G, axis=-1), 1, axis=-1)
        assert np.array_equal(G, Gm)  # conjugate pairs share the multiplier (Eq 16)
        P = greens.dense_P_mixed2d(G, g.node_shape)
    ok, lo, _ = greens.eq55_check(np.concatenate([np.zeros((c, c, 1)), G.reshape(c, c, -1)], axis=-1))
    assert ok and lo > 0
    ev = np.sort(np.linalg.eigvalsh(P))
    evb = np.sort(np.linalg.eigvalsh(np.moveaxis(G.reshape(c, c, -1), -1, 0)).reshape(-1))
    assert np.max(np.abs(ev - evb)) < 1e-9 * evb.max()


@pytest.mark.parametrize("bc", [(1, 1), (0, 1)])
@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_pcg_vs_dense_solve(bc, physics):
    c = 1 if physics == "thermal" else 2
    g = fem.Grid((8, 6), bc=bc, c=c)
    ph = (RNG.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 20.0) if c == 1 else ((0.58, 0.38), (2.78, 4.17))
    load = np.eye(2 if c == 1 else 3)[0]
    out = homog.solve_problem(g, physics, ph, mat, [load], 9, 0.1 if c == 1 else 0.05, tol=1e-12)
    A = fem.assemble_dense(g, physics, ph, mat)
    f = fem.rhs(g, physics, ph, mat, load)
    x = np.linalg.solve(A, f.reshape(-1)).reshape(f.shape)
    assert out["results"][0].converged
    assert np.linalg.norm(out["U"][0] - x) <= 1e-9 * np.linalg.norm(x)
