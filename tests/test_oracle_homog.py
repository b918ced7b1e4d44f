"""Pins for oracle/homog.py (not gpu): homogeneous medium, laminates (Voigt/Reuss and the
elastic layer-averaging closed form), effective-property identities and bounds.
SURVEY §8(c) C4; §5 (Eq 74-84), App. A."""
import numpy as np
import pytest

from oracle import fem, greens, homog, pcg
from paper_2508_02681_b200 import synth

RNG = np.random.default_rng(99)


def test_homogeneous_thermal_and_elastic():
    g = fem.Grid((6, 6, 6))
    ph = np.zeros(g.elem_shape, np.uint8)
    out = homog.solve_problem(g, "thermal", ph, (2.5, 7.0), np.eye(3), 5, 0.1)
    assert out["iterations"] == [0, 0, 0]
    assert np.max(np.abs(out["effective"] - 2.5 * np.eye(3))) < 1e-14
    g3 = fem.Grid((4, 4, 4), c=3)
    mat = ((0.6, 0.4), (3.0, 2.0))
    out = homog.solve_problem(g3, "elastic", np.zeros(g3.elem_shape, np.uint8), mat, np.eye(6), 5, 0.05)
    assert out["iterations"] == [0] * 6
    assert np.max(np.abs(out["effective"] - fem.isotropic_D(3, 0.6, 0.4))) < 1e-14


@pytest.mark.parametrize("normal", [0, 1, 2])
def test_thermal_laminate_voigt_reuss(normal):
    N = (8, 8, 8)
    g = fem.Grid(N)
    ph = synth.laminate(g.elem_shape, normal, period=4, width=1)
    k0, k1 = 1.0, 10.0
    vf = ph.mean()
    out = homog.solve_problem(g, "thermal", ph, (k0, k1), np.eye(3), 3, 0.1, tol=1e-13)
    voigt, reuss = homog.voigt_reuss(k0, k1, vf)
    expect = voigt * np.eye(3)
    expect[normal, normal] = reuss
    assert np.max(np.abs(out["effective"] - expect)) < 1e-11


@pytest.mark.parametrize("normal", [0, 2])
def test_elastic_laminate_closed_form(normal):
    N = (4, 4, 8) if normal == 2 else (8, 4, 4)
    g = fem.Grid(N, c=3)
    ph = synth.laminate(g.elem_shape, normal, period=4, width=1)
    mat = ((0.58, 0.38), (2.78, 4.17))
    vf = ph.mean()
    out = homog.solve_problem(g, "elastic", ph, mat, np.eye(6), 3, 0.05, tol=1e-13)
    D0, D1 = fem.isotropic_D(3, *mat[0]), fem.isotropic_D(3, *mat[1])
    for j in range(6):
        sig = homog.laminate_elastic(3, normal, D0, D1, vf, np.eye(6)[j])
        assert np.max(np.abs(out["effective"][:, j] - sig)) < 1e-10


def test_effective_identities_and_bounds():
    P = synth.config0()
    g = fem.Grid((32, 32))
    out = homog.solve_problem(g, "thermal", P.phase, P.mat, np.eye(2), P.seed, 0.1, tol=1e-12)
    K = out["effective"]
    assert abs(K[0, 1] - K[1, 0]) < 1e-9 * K[0, 0]                       # symmetry
    for j in range(2):                                                    # centroid-flux identity
        avg = homog.centroid_flux_average(g, P.phase, P.mat, np.eye(2)[j], out["U"][j])
        assert np.max(np.abs(avg - K[:, j])) < 1e-9
    vf = P.phase.mean()
    voigt, reuss = homog.voigt_reuss(*P.mat, vf)
    lo, hi = homog.hs_thermal(*P.mat, vf, d=2)
    for i in range(2):
        assert reuss <= K[i, i] <= voigt
        assert lo - 0.05 <= K[i, i] <= hi + 0.05                          # HS (soft: finite sample)


def test_diagonal_quadratic_convergence_galerkin():
    # f.u_m = u_m.K u_m for CG iterates from u0 = 0 (Galerkin orthogonality)
    g = fem.Grid((8, 8, 8))
    ph = (RNG.random(g.elem_shape) < 0.3).astype(np.uint8)
    mat = (1.0, 50.0)
    f = fem.rhs(g, "thermal", ph, mat, np.eye(3)[0])
    G = greens.ghat(g, "thermal", mat, 3, 0.1)
    for m in (1, 3, 6):
        u = pcg.pcg(lambda v: fem.apply_K(g, "thermal", ph, mat, v), lambda v: greens.apply_precond(G, v), f,
                    fixed_iters=m).u
        assert abs(np.sum(f * u) - np.sum(u * fem.apply_K(g, "thermal", ph, mat, u))) < 1e-12 * abs(np.sum(f * u))
