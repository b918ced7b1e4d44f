"""Pins for oracle/fem.py against closed forms, invariants and brute force (not gpu).

PAPER.md §3.1 Eq 22; SURVEY §8(c) C4 rows 'Element matrices',
'Assembled stencil', 'K symmetry/PSD', 'K vs assembled', 'RHS'.
"""
import itertools
import math

import numpy as np
import pytest

from oracle import fem

RNG = np.random.default_rng(1234)


def test_thermal_element_2d_closed_form():
    # SPEC S:108 "diagonal entries 2/3"; {2/3 diag, -1/6 edge, -1/3 diagonal}.
    K = fem.element_stiffness_thermal(2, (1.0, 1.0))
    cs = fem.corners(2)
    for i, a in enumerate(cs):
        for j, b in enumerate(cs):
            ham = sum(x != y for x, y in zip(a, b))
            expect = {0: 2 / 3, 1: -1 / 6, 2: -1 / 3}[ham]
            assert abs(K[i, j] - expect) < 1e-15
    # h-independence in 2D
    assert np.allclose(fem.element_stiffness_thermal(2, (0.25, 0.25)), K, atol=1e-15)


def test_thermal_element_3d_tensor_form():
    # App. A1: K = sum_i k_i (x) m_j (x) m_l with k = (1/h)[[1,-1],[-1,1]], m = (h/6)[[2,1],[1,2]].
    h = 0.125
    k = np.array([[1, -1], [-1, 1]]) / h
    m = np.array([[2, 1], [1, 2]]) * h / 6
    # corner index a_x + 2 a_y + 4 a_z -> kron order (z, y, x)
    T = np.kron(np.kron(m, m), k) + np.kron(np.kron(m, k), m) + np.kron(np.kron(k, m), m)
    K = fem.element_stiffness_thermal(3, (h, h, h))
    assert np.max(np.abs(K - T)) < 1e-15
    # closed-form values h*{1/3, 0, -1/12, -1/12}
    cs = fem.corners(3)
    for i, a in enumerate(cs):
        for j, b in enumerate(cs):
            ham = sum(x != y for x, y in zip(a, b))
            assert abs(K[i, j] - h * {0: 1 / 3, 1: 0.0, 2: -1 / 12, 3: -1 / 12}[ham]) < 1e-15


@pytest.mark.parametrize("d", [2, 3])
def test_elastic_element_patch_and_rigid_modes(d):
    h = tuple(0.5 + 0.25 * i for i in range(d))  # anisotropic voxel on purpose
    Kl, Km = fem.element_stiffness_elastic(d, h)
    lam, mu = 0.7, 1.3
    Ke = lam * Kl + mu * Km
    assert np.max(np.abs(Ke - Ke.T)) < 1e-14
    cs = fem.corners(d)
    X = np.array([[a[i] * h[i] for i in range(d)] for a in cs])
    # rigid translations and infinitesimal rotations are in the null space
    ev = np.linalg.eigvalsh(Ke)
    nrigid = d + d * (d - 1) // 2
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == nrigid
    # patch test: affine field u = E x  =>  u^T K u = vol * eps : D : eps  (Q1 exact for affine)
    for _ in range(5):
        E = RNG.standard_normal((d, d))
        u = (X @ E.T).reshape(-1)  # dof order (corner, component)
        eps = 0.5 * (E + E.T)
        sig = lam * np.trace(eps) * np.eye(d) + 2 * mu * eps
        assert abs(u @ Ke @ u - np.prod(h) * np.sum(sig * eps)) < 1e-12 * max(1, abs(u @ Ke @ u))


def test_homogeneous_stencil_3d():
    # 8/3 h centre, 0 axis, -h/6 face diagonal, -h/12 corner; row sum 0.
    n = 6
    g = fem.Grid((n, n, n))
    h = 1.0 / n
    d = np.zeros((1, n, n, n))
    d[0, 0, 0, 0] = 1.0
    s = fem.apply_K_thermal(g, np.zeros((n, n, n), np.uint8), (1.0, 1.0), d)[0]
    for off in itertools.product((-1, 0, 1), repeat=3):
        nz = sum(o != 0 for o in off)
        expect = h * {0: 8 / 3, 1: 0.0, 2: -1 / 6, 3: -1 / 12}[nz]
        assert abs(s[off[2] % n, off[1] % n, off[0] % n] - expect) < 1e-15
    assert abs(s.sum()) < 1e-14


def test_jacobi_diagonal_2d_dirichlet():
    # homogeneous kappa=1, interior node of a Dirichlet 2D grid: 1/A_ii = 3/8.
    g = fem.Grid((5, 5), bc=(1, 1))
    A = fem.assemble_dense(g, "thermal", np.zeros((5, 5), np.uint8), (1.0, 1.0))
    assert np.allclose(1.0 / np.diag(A), 3 / 8, atol=1e-15)


CASES = [
    ((4, 3, 5), (0, 0, 0)), ((4, 3, 5), (0, 0, 1)), ((3, 4, 3), (1, 1, 1)),
    ((5, 4), (0, 0)), ((4, 5), (0, 1)), ((4, 4), (1, 1)),
]


@pytest.mark.parametrize("N,bc", CASES)
@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_matrix_free_equals_dense_assembly(N, bc, physics):
    d = len(N)
    c = 1 if physics == "thermal" else d
    g = fem.Grid(N, bc=bc, c=c)
    ph = (RNG.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 7.0) if physics == "thermal" else ((0.5, 0.3), (2.0, 4.0))
    A = fem.assemble_dense(g, physics, ph, mat)
    assert np.max(np.abs(A - A.T)) < 1e-13                       # symmetry
    ev = np.linalg.eigvalsh(A)
    assert ev.min() > -1e-12 * ev.max()                          # PSD
    if all(b == 1 for b in bc):
        assert ev.min() > 0                                      # Dirichlet: SPD
    for _ in range(3):
        u = RNG.standard_normal(g.field_shape())
        Ku = fem.apply_K(g, physics, ph, mat, u)
        assert np.max(np.abs(A @ u.reshape(-1) - Ku.reshape(-1))) < 1e-12 * max(1, np.abs(A).max())


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_periodic_nullspace_per_component(physics):
    g = fem.Grid((6, 5, 4), c=1 if physics == "thermal" else 3)
    ph = (RNG.random(g.elem_shape) < 0.5).astype(np.uint8)
    mat = (1.0, 30.0) if physics == "thermal" else ((0.5, 0.3), (5.0, 8.0))
    for comp in range(g.c):
        u = np.zeros(g.field_shape())
        u[comp] = 1.0
        assert np.max(np.abs(fem.apply_K(g, physics, ph, mat, u))) < 1e-13


def _affine_rhs_via_element_matrices(g, physics, phase, mat, load):
    """Independent route: f = -sum_e scatter(K_e u_e^aff), u^aff = gbar.x (thermal) or
    eps_bar.x (elastic) evaluated at the element's local corner coordinates."""
    d = g.d
    cs = fem.corners(d)
    X = np.array([[a[i] * g.h[i] for i in range(d)] for a in cs])
    uf = fem._pad_full(g, np.zeros(g.field_shape()))
    out = np.zeros_like(uf)
    if physics == "thermal":
        Kr = fem.element_stiffness_thermal(d, g.h)
        ue = X @ np.asarray(load)
        coef = fem.coeff_field(phase, *mat)[None]
        for ai, a in enumerate(cs):
            fem._scatter_add(g, out, -coef * float(Kr[ai] @ ue), a)
    else:
        Kl, Km = fem.element_stiffness_elastic(d, g.h)
        pairs = fem._mandel_pairs(d)
        E = np.zeros((d, d))
        for mi, (i, j) in enumerate(pairs):
            if i == j:
                E[i, i] = load[mi]
            else:
                E[i, j] = E[j, i] = load[mi] / math.sqrt(2)
        ue = (X @ E.T).reshape(-1)
        (l0, m0), (l1, m1) = mat
        lam = fem.coeff_field(phase, l0, l1)
        mu = fem.coeff_field(phase, m0, m1)
        vl, vm = Kl @ ue, Km @ ue
        for ai, a in enumerate(cs):
            v = np.stack([-(lam * vl[d * ai + al] + mu * vm[d * ai + al]) for al in range(d)])
            fem._scatter_add(g, out, v, a)
    return fem._interior(g, out)


@pytest.mark.parametrize("bc", [(0, 0, 0), (0, 0, 1)])
@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_rhs(physics, bc):
    d = 3
    g = fem.Grid((5, 4, 6), bc=bc, c=1 if physics == "thermal" else 3)
    ph = (RNG.random(g.elem_shape) < 0.35).astype(np.uint8)
    mat = (1.0, 10.0) if physics == "thermal" else ((0.6, 0.4), (2.8, 4.2))
    nl = 3 if physics == "thermal" else 6
    for j in range(nl):
        load = np.eye(nl)[j]
        f = fem.rhs(g, physics, ph, mat, load)
        f2 = _affine_rhs_via_element_matrices(g, physics, ph, mat, load)
        assert np.max(np.abs(f - f2)) < 1e-14
        if bc == (0, 0, 0):
            assert np.max(np.abs(f.sum(axis=tuple(range(1, f.ndim))))) < 1e-13
        # homogeneous medium => f = 0 (periodic)
        if bc == (0, 0, 0):
            f0 = fem.rhs(g, physics, np.zeros_like(ph), mat, load)
            assert np.max(np.abs(f0)) < 1e-14
    # linear in the load
    a = RNG.standard_normal(nl)
    fa = fem.rhs(g, physics, ph, mat, a)
    fs = sum(a[j] * fem.rhs(g, physics, ph, mat, np.eye(nl)[j]) for j in range(nl))
    assert np.max(np.abs(fa - fs)) < 1e-13


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_apply_K_at_equals_full_apply(physics):
    # sampled-output evaluator used by the full-size GPU tests == full matrix-free apply
    c = 1 if physics == "thermal" else 3
    g = fem.Grid((8, 6, 10), c=c, h=1 / 8)
    ph = (RNG.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 9.0) if physics == "thermal" else ((0.5, 0.3), (2.0, 4.0))
    u = RNG.standard_normal(g.field_shape())
    K = fem.apply_K(g, physics, ph, mat, u)
    nodes = [(0, 0, 0), (9, 5, 7), (4, 2, 3), (9, 0, 7)]
    got = fem.apply_K_at(g, physics, ph, mat, u, nodes)
    assert np.max(np.abs(got - np.array([K[(slice(None),) + n] for n in nodes]))) < 1e-14


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
@pytest.mark.parametrize("bc", [(0, 0, 0), (0, 0, 1), (1, 1, 1)])
@pytest.mark.parametrize("zchunk,workers", [(1, 1), (3, 2), (64, 1)])
def test_chunked_K_equals_K(physics, bc, zchunk, workers):
    # the slab evaluation used for the 256^3 / 512^3 goldens is apply_K exactly
    g = fem.Grid((6, 4, 8), bc=bc, c=1 if physics == "thermal" else 3, h=0.125)
    rng = np.random.default_rng(5)
    ph = (rng.random(g.elem_shape) < 0.4).astype(np.uint8)
    mat = (1.0, 7.0) if physics == "thermal" else ((0.6, 0.4), (2.8, 4.2))
    u = rng.standard_normal(g.field_shape())
    ref = fem.apply_K(g, physics, ph, mat, u)
    got = fem.apply_K_chunked(g, physics, ph, mat, u, zchunk=zchunk, workers=workers)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
