"""Pins for oracle/transform.py and oracle/greens.py (not gpu).

SURVEY §8(c) C4 rows 'Transform', 'G_hat vs K', 'P properties', 'Lemma 1',
'FANS spectrum', 'Perturbation'; Eq 47-55, Lemma 1 / App. C, Tab 4.
"""
import json
import os

import numpy as np
import pytest

from oracle import fem, greens, pcg, transform

RNG = np.random.default_rng(42)
GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- transform
@pytest.mark.parametrize("shape", [(4,), (6, 4), (3, 4, 5)])
def test_dense_T_unitary_and_matches_forward(shape):
    T = transform.dense_T(shape)
    n = int(np.prod(shape))
    assert np.max(np.abs(T.conj().T @ T - np.eye(n))) < 1e-13
    x = RNG.standard_normal(shape)
    full = np.fft.fftn(x, norm="ortho").reshape(-1)
    assert np.max(np.abs(T @ x.reshape(-1) - full)) < 1e-13
    xh = transform.forward(x[None])[0]
    assert np.max(np.abs(xh - full.reshape(shape)[..., : shape[-1] // 2 + 1])) < 1e-13
    assert abs(np.linalg.norm(T @ x.reshape(-1)) - np.linalg.norm(x)) < 1e-12
    y = transform.inverse(transform.forward(x[None]), shape)[0]
    assert np.max(np.abs(y - x)) < 1e-13


def test_zero_frequency_impulse():
    # inverse of the zero-frequency impulse -> constant 1/sqrt(n)
    shape = (4, 6, 8)
    rh = np.zeros((1, 4, 6, 5), complex)
    rh[0, 0, 0, 0] = 1.0
    x = transform.inverse(rh, shape)
    assert np.max(np.abs(x - 1 / np.sqrt(4 * 6 * 8))) < 1e-15


def test_parseval_weights():
    for shape in [(8, 6), (4, 4, 8), (5, 7)]:
        a, b = RNG.standard_normal(shape), RNG.standard_normal(shape)
        ah, bh = transform.forward(a[None])[0], transform.forward(b[None])[0]
        s = np.sum(transform.parseval_weights(shape) * (np.conj(ah) * bh).real)
        assert abs(s - np.sum(a * b)) < 1e-12


# ----------------------------------------------------------------------------- symbol
def _closed_form_symbol(N, h, physics, ref):
    """SURVEY App. A3 closed forms (theta_i = 2 pi k_i / N_i), numpy axis order."""
    d = len(N)
    grids = np.meshgrid(*[2 * np.pi * np.arange(N[i]) / N[i] for i in reversed(range(d))], indexing="ij")
    th = list(reversed(grids))  # th[i] for physical axis i
    mass = [(h[i] / 3) * (2 + np.cos(th[i])) for i in range(d)]
    S = np.zeros((d, d) + grids[0].shape)
    for i in range(d):
        v = (2 / h[i]) * (1 - np.cos(th[i]))
        for j in range(d):
            if j != i:
                v = v * mass[j]
        S[i, i] = v
        for j in range(d):
            if j != i:
                w = np.sin(th[i]) * np.sin(th[j])
                for l in range(d):
                    if l not in (i, j):
                        w = w * mass[l]
                S[i, j] = w
    if physics == "thermal":
        return ref * np.trace(S)[None, None]
    lam, mu = ref
    tr = np.trace(S)
    return (lam + mu) * S + mu * np.einsum("ij,...->ij...", np.eye(d), tr)


@pytest.mark.parametrize("N", [(8, 6, 4), (16, 8), (6, 6, 6)])
@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_probe_symbol_matches_closed_form(N, physics):
    d = len(N)
    g = fem.Grid(N, c=1 if physics == "thermal" else d)
    ref = 1.7 if physics == "thermal" else (1.6774, 2.2756)
    A = greens.symbol_probe(g, physics, ref)
    C = _closed_form_symbol(N, g.h, physics, ref)
    assert np.max(np.abs(A - C)) < 1e-13 * max(1.0, np.abs(C).max())


def test_homogeneous_PK_is_identity_minus_mean():
    # Key joint pin: homogeneous medium, seed 0 => P K u = u - mean(u) per component.
    for physics, c, mat in [("thermal", 1, (2.5, 2.5)), ("elastic", 3, ((0.9, 0.5), (0.9, 0.5))),
                            ("elastic", 2, ((0.9, 0.5), (0.9, 0.5)))]:
        N = (8, 6, 4) if c != 2 else (8, 6)
        g = fem.Grid(N, c=c)
        ph = np.zeros(g.elem_shape, np.uint8)
        G = greens.ghat(g, physics, mat, 0, 0.0)
        u = RNG.standard_normal(g.field_shape())
        v = greens.apply_precond(G, fem.apply_K(g, physics, ph, mat, u))
        assert np.max(np.abs(v - pcg.remove_mean(u))) < 1e-12


@pytest.mark.parametrize("physics,N", [("thermal", (8, 6, 4)), ("thermal", (16, 16)), ("elastic", (6, 4, 8))])
def test_perturbed_symbol_invariants(physics, N):
    d = len(N)
    g = fem.Grid(N, c=1 if physics == "thermal" else d)
    mat = (1.0, 10.0) if physics == "thermal" else ((0.58, 0.38), (2.78, 4.17))
    amp = 0.1 if physics == "thermal" else 0.05
    G = greens.ghat(g, physics, mat, 77, amp)
    # G(-k) == G(k) bit-exactly (Eq 16)
    Gm = G
    for ax in range(2, G.ndim):
        Gm = np.roll(np.flip(Gm, axis=ax), 1, axis=ax)
    assert np.array_equal(G, Gm)
    ok, lo, hi = greens.eq55_check(G)  # Eq 55
    assert ok and lo > 0
    assert np.all(G[(slice(None), slice(None)) + (0,) * d] == 0)
    G0 = greens.ghat(g, physics, mat, 0, amp)
    if physics == "thermal":
        nz = G0 != 0
        rho = G[nz] / G0[nz]
        assert rho.min() >= 1 - amp - 1e-15 and rho.max() <= 1 + amp + 1e-15
        assert rho.std() > 0.02  # actually perturbed
    else:
        # G - Phi = amp tr(Phi)/3 psi is PSD (psi = L L^T, Eq B5)
        D = np.moveaxis((G - G0).reshape(d, d, -1), -1, 0)
        assert np.linalg.eigvalsh(D).min() > -1e-14


def test_psi3_is_LLt():
    th = RNG.standard_normal((6, 50))
    P = greens.psi3(th)
    for k in range(50):
        t1, t2, t3, t4, t5, t6 = th[:, k]
        L = np.array([[t1, 0, 0], [t3, t2, 0], [t6, t5, t4]])
        assert np.max(np.abs(P[:, :, k] - L @ L.T)) < 1e-14


# ----------------------------------------------------------------------------- P properties
def _random_consistent_symbol(shape, c):
    """Random SPD blocks that depend only on the pair {k,-k}."""
    can = greens.canon_index(shape).reshape(-1)
    n = can.size
    B = RNG.standard_normal((n, c, c))
    blocks = np.einsum("nij,nkj->nik", B, B) + 0.1 * np.eye(c)
    blocks = blocks[can]  # consistent under k -> -k
    return np.moveaxis(blocks, 0, -1).reshape((c, c) + tuple(shape))


@pytest.mark.parametrize("shape,c", [((6, 6), 1), ((4, 4), 2), ((4, 2, 4), 3), ((5, 4), 1)])
def test_lemma1_bruteforce(shape, c):
    # Lemma 1 (App. C): eig(T^H Q T) = union_k eig(Phi(k)).
    for _ in range(3):
        G = _random_consistent_symbol(shape, c)
        P = greens.dense_P(G, shape)
        assert np.max(np.abs(P - P.T)) < 1e-12
        ev = np.sort(np.linalg.eigvalsh(P))
        blocks = np.moveaxis(G.reshape(c, c, -1), -1, 0)
        evb = np.sort(np.linalg.eigvalsh(blocks).reshape(-1))
        assert np.max(np.abs(ev - evb)) < 1e-9 * max(1, evb.max())
        # fast apply == dense Eq 48 matrix
        r = RNG.standard_normal((c,) + shape)
        s = greens.apply_precond(G, r)
        assert np.max(np.abs(s.reshape(-1) - P @ r.reshape(-1))) < 1e-12
        assert abs(greens.gamma_parseval(G, r) - float(np.sum(r * s))) < 1e-11 * abs(np.sum(r * s))


def test_precond_A1_A2_A3():
    # [A1]-[A3] on the perturbed elastic symbol
    g = fem.Grid((6, 4, 8), c=3)
    G = greens.ghat(g, "elastic", ((0.58, 0.38), (2.78, 4.17)), 5, 0.05)
    r1, r2 = RNG.standard_normal(g.field_shape()), RNG.standard_normal(g.field_shape())
    a = 0.37
    s12 = greens.apply_precond(G, a * r1 + r2)
    assert np.max(np.abs(s12 - (a * greens.apply_precond(G, r1) + greens.apply_precond(G, r2)))) < 1e-13
    x = np.sum(r1 * greens.apply_precond(G, r2))
    y = np.sum(r2 * greens.apply_precond(G, r1))
    assert abs(x - y) < 1e-12 * max(abs(x), 1)
    for _ in range(5):
        r = pcg.remove_mean(RNG.standard_normal(g.field_shape()))
        assert np.sum(r * greens.apply_precond(G, r)) > 0


def test_fans_spectrum_table4_bounds():
    # Tab 4 FANS row: lambda in [1/3, 5/3], cond 5 for kappa 1/0.2, kappa_r = 0.6.
    # SPEC acceptance 1: 32^2 random microstructure.
    tab = json.load(open(os.path.join(GOLD, "table4.json")))
    fans = [r for r in tab["rows"] if r["solver"] == "FANS"][0]
    N = (32, 32)
    g = fem.Grid(N)
    ph = (RNG.random(g.elem_shape) < 0.5).astype(np.uint8)
    mat = (tab["fans_material"]["kappa0"], tab["fans_material"]["kappa1"])
    A = fem.assemble_dense(g, "thermal", ph, mat)
    G = greens.ghat(g, "thermal", mat, 0, 0.0)
    P = greens.dense_P(G, N)
    ev = np.sort(np.linalg.eigvals(P @ A).real)[1:]  # drop the shared constant null mode
    assert ev.min() >= 1 / 3 - 1e-10 and ev.max() <= 5 / 3 + 1e-10
    assert abs(ev.min() - fans["lmin"]) < 0.01 and abs(ev.max() - fans["lmax"]) < 0.04
    assert 4.9 <= ev.max() / ev.min() <= 5.2
    # with the seeded rho in [0.9, 1.1] the bound widens to [0.9/3, 1.1*5/3]
    Gp = greens.ghat(g, "thermal", mat, 9, 0.1)
    evp = np.sort(np.linalg.eigvals(greens.dense_P(Gp, N) @ A).real)[1:]
    assert evp.min() >= 0.9 / 3 - 1e-10 and evp.max() <= 1.1 * 5 / 3 + 1e-10


# ----------------------------------------------------------------------------- long axes
def _closed_form_symbol_stable(N, h, physics, ref):
    """SURVEY App. A3 closed forms with 1 - cos(t) written as 2 sin^2(t/2) (no cancellation at low
    frequency), signed frequencies; an independent route to the symbol on 512-1024-point axes."""
    d = len(N)
    grids = np.meshgrid(*[2 * np.pi * np.fft.fftfreq(N[i]) for i in reversed(range(d))], indexing="ij")
    th = list(reversed(grids))
    mass = [(h[i] / 3) * (2 + np.cos(th[i])) for i in range(d)]
    S = np.zeros((d, d) + grids[0].shape)
    for i in range(d):
        v = (4 / h[i]) * np.sin(th[i] / 2) ** 2
        for j in range(d):
            if j != i:
                v = v * mass[j]
        S[i, i] = v
        for j in range(d):
            if j != i:
                w = np.sin(th[i]) * np.sin(th[j])
                for l in range(d):
                    if l not in (i, j):
                        w = w * mass[l]
                S[i, j] = w
    if physics == "thermal":
        return ref * np.trace(S)[None, None]
    lam, mu = ref
    return (lam + mu) * S + mu * np.einsum("ij,...->ij...", np.eye(d), np.trace(S))


@pytest.mark.parametrize("N,physics", [((1024, 8, 4), "thermal"), ((4, 1024, 8), "elastic"),
                                       ((8, 4, 512), "elastic"), ((1024, 512), "thermal")])
def test_symbol_relative_accuracy_on_long_axes(N, physics):
    # the stencil DFT is evaluated without cancellation: every bin, including the lowest
    # frequencies of a 512-1024-point axis (symbol ~ theta^2 ~ 4e-5), to ~1e-15 relative
    d = len(N)
    g = fem.Grid(N, c=1 if physics == "thermal" else d, h=1.0 / max(N))
    ref = 1.7 if physics == "thermal" else (1.6774, 2.2756)
    A = greens.symbol_probe(g, physics, ref)
    C = _closed_form_symbol_stable(N, g.h, physics, ref)
    nrm = np.sqrt(np.sum(C ** 2, axis=(0, 1)))
    err = np.sqrt(np.sum((A - C) ** 2, axis=(0, 1)))
    nz = nrm > 0
    assert np.count_nonzero(~nz) == 1 and np.all(A[(slice(None), slice(None)) + (0,) * d] == 0)
    assert np.max(err[nz] / nrm[nz]) < 1e-14


@pytest.mark.parametrize("physics,N", [("thermal", (16, 8, 6)), ("elastic", (8, 6, 10)), ("elastic", (12, 8))])
def test_half_spectrum_and_chunked_symbol_equal_full(physics, N):
    # ghat(half=True) is the R2C restriction of the full table, chunking changes nothing
    d = len(N)
    g = fem.Grid(N, c=1 if physics == "thermal" else d)
    mat = (1.0, 10.0) if physics == "thermal" else ((0.58, 0.38), (2.78, 4.17))
    G = greens.ghat(g, physics, mat, 77, 0.1)
    Gh = greens.ghat(g, physics, mat, 77, 0.1, half=True, zchunk=3)
    assert np.array_equal(Gh, greens.half(G))
    assert np.array_equal(greens.ghat(g, physics, mat, 77, 0.1, zchunk=1), G)
    r = RNG.standard_normal(g.field_shape())
    assert np.max(np.abs(greens.apply_precond(Gh, r) - greens.apply_precond(G, r))) == 0.0
