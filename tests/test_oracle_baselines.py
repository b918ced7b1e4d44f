"""Pins for oracle/baselines.py (P = I and Jacobi, Eq 25): diag(A) against the
diagonal of the dense assembly (brute force) and SPEC S:140's closed form; Jacobi on a
homogeneous medium is a scaled identity, so PCG iterates equal unpreconditioned CG's
(scale invariance of PCG).  Not gpu."""
import numpy as np
import pytest

from oracle import baselines, fem, pcg

RNG = np.random.default_rng(77)

CASES = [((4, 3, 5), (0, 0, 0)), ((4, 3, 5), (0, 0, 1)), ((3, 4, 3), (1, 1, 1)), ((5, 4), (0, 0)), ((4, 4), (1, 1))]


@pytest.mark.parametrize("N,bc", CASES)
@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_diag_equals_dense_assembly(N, bc, physics):
    d = len(N)
    g = fem.Grid(N, bc=bc, c=1 if physics == "thermal" else d)
    ph = (RNG.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 7.0) if physics == "thermal" else ((0.5, 0.3), (2.0, 4.0))
    A = fem.assemble_dense(g, physics, ph, mat)
    dg = baselines.diag_K(g, physics, ph, mat)
    assert np.max(np.abs(dg.reshape(-1) - np.diag(A))) < 1e-13 * np.abs(A).max()


def test_jacobi_closed_form_2d_dirichlet():
    # homogeneous kappa = 1, 2D Dirichlet grid: 1/A_ii = 3/8 at every free node
    g = fem.Grid((5, 5), bc=(1, 1))
    dg = baselines.diag_K(g, "thermal", np.zeros((5, 5), np.uint8), (1.0, 1.0))
    assert np.allclose(1.0 / dg, 3 / 8, atol=1e-15)


def test_closed_form_diagonals_3d():
    # every Q1 corner has the same element diagonal: thermal h/3, elastic lam h/9 + mu 4h/9
    h = 1 / 6
    g = fem.Grid((6, 4, 4), h=h)
    ph = (RNG.random(g.elem_shape) < 0.5).astype(np.uint8)
    n1 = sum(np.roll(np.roll(np.roll(ph, ox, 2), oy, 1), oz, 0) for ox in (0, 1) for oy in (0, 1) for oz in (0, 1))
    dt = baselines.diag_K(g, "thermal", ph, (2.0, 9.0))[0]
    assert np.max(np.abs(dt - h / 3 * ((8 - n1) * 2.0 + n1 * 9.0))) < 1e-14
    ge = fem.Grid((6, 4, 4), c=3, h=h)
    de = baselines.diag_K(ge, "elastic", ph, ((0.5, 0.3), (2.0, 4.0)))
    e0, e1 = h / 9 * (0.5 + 4 * 0.3), h / 9 * (2.0 + 4 * 4.0)
    for al in range(3):
        assert np.max(np.abs(de[al] - ((8 - n1) * e0 + n1 * e1))) < 1e-14


def test_jacobi_on_homogeneous_medium_is_scaled_cg():
    g = fem.Grid((6, 5, 4), h=1 / 6)
    ph = np.zeros(g.elem_shape, np.uint8)
    f = RNG.standard_normal(g.field_shape())
    f -= f.mean()
    A = lambda v: fem.apply_K(g, "thermal", ph, (3.0, 3.0), v)  # noqa: E731
    dg = baselines.diag_K(g, "thermal", ph, (3.0, 3.0))
    assert np.ptp(dg) == 0.0
    a = pcg.pcg(A, lambda r: r / dg, f, fixed_iters=8)
    b = pcg.pcg(A, lambda r: r.copy(), f, fixed_iters=8)
    assert np.max(np.abs(a.u - b.u)) < 1e-12 * np.abs(b.u).max()
