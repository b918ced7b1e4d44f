"""Preconditioner symbol G_hat and the UNO apply — oracle (TEST INFRASTRUCTURE ONLY).

* FANS reference-medium operator (§3.3.4, Eq 33-37): A_r is
  block circulant, so P_FANS = F^{-1} Phi_hat F with Phi_hat(k) the
  (pseudo-)inverse of the Fourier symbol A_r_hat(k).  "Assembled ... by solving an
  auxiliary linear system": here the symbol is obtained by PROBING the
  matrix-free reference stiffness with a unit impulse per component and taking
  its DFT (convolution theorem).
* No trained UNO weights exist (BASELINE.json north_star), so
  G_hat = FANS symbol x seeded SPD perturbation:
    c = 1:  G_hat(k) = rho(k) / A_r_hat(k),  rho = 1 - amp + 2 amp u01(seed, 2, canon(k))
    c = 3:  G_hat(k) = Phi_hat(k) + amp (tr Phi_hat(k)/3) psi(theta(k)),  psi = Eq B5
  with the multiplier a function of the unordered pair {k, -k} (Eq 16, P:187;
  SURVEY A9) and G_hat(0) = 0 (null space shared with periodic K).
* UNO apply: s = T^H Q T r (Eq 46-49), Q block diagonal per frequency.
* Eq 55 safety check over all blocks k != 0.

The perturbation's random numbers use this module's own SplitMix64 (the CUDA
library implements the same counter-based generator independently).
"""
from __future__ import annotations

import numpy as np

from . import fem, transform

_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _sm64(x):
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + _GOLD
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def u01(seed: int, stream: int, idx) -> np.ndarray:
    """Counter-based uniform in [0,1): (sm64(seed ^ sm64(stream ^ sm64(i))) >> 11) 2^-53."""
    v = _sm64(np.uint64(seed) ^ _sm64(np.uint64(stream) ^ _sm64(idx)))
    return (v >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def reference_medium(physics: str, mat):
    """Arithmetic mean of the phase parameters."""
    if physics == "thermal":
        return 0.5 * (mat[0] + mat[1])
    (l0, m0), (l1, m1) = mat
    return (0.5 * (l0 + l1), 0.5 * (m0 + m1))


def symbol_probe(g: fem.Grid, physics: str, ref) -> np.ndarray:
    """A_r_hat(k) by probing the homogeneous reference stiffness (periodic grid).
    Returns the full spectrum: shape (c, c) + spatial (real; imaginary part ~ 1e-16)."""
    assert all(b == 0 for b in g.bc), "FANS symbol needs a periodic grid (P:470)"
    c = g.c
    shp = g.node_shape
    phase0 = np.zeros(g.elem_shape, dtype=np.uint8)
    mat = (ref, ref) if physics == "thermal" else (ref, ref)
    out = np.zeros((c, c) + shp, dtype=complex)
    for b in range(c):
        delta = np.zeros((c,) + shp)
        delta[(b,) + (0,) * len(shp)] = 1.0
        col = fem.apply_K(g, physics, phase0, mat, delta)  # column b of the stencil
        for a in range(c):
            out[a, b] = np.fft.fftn(col[a])
    assert np.max(np.abs(out.imag)) < 1e-9 * max(1.0, np.max(np.abs(out.real)))
    A = out.real
    # K real symmetric => A_hat(k) real symmetric and A_hat(-k) = A_hat(k) exactly; remove the
    # FFT round-off asymmetry so the multiplier is a function of {k,-k} bit-exactly (Eq 16).
    Am = A
    for ax in range(2, A.ndim):
        Am = np.roll(np.flip(Am, axis=ax), 1, axis=ax)
    A = 0.5 * (A + Am)
    A = 0.5 * (A + np.swapaxes(A, 0, 1))
    return A.copy()


def canon_index(shape) -> np.ndarray:
    """canon(k) = min(flat(k), flat(-k mod N)) over the full frequency grid (C order,
    x fastest) — the unordered pair {k, -k}."""
    grids = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    flat = np.zeros(shape, dtype=np.int64)
    flatn = np.zeros(shape, dtype=np.int64)
    for ax, n in enumerate(shape):
        flat = flat * n + grids[ax]
        flatn = flatn * n + ((-grids[ax]) % n)
    return np.minimum(flat, flatn)


def psi3(th: np.ndarray) -> np.ndarray:
    """Local SPD parametrisation for c = 3, Eq B5.  th: (6, ...) -> (3, 3, ...)."""
    t1, t2, t3, t4, t5, t6 = th
    return np.array([
        [t1 * t1, t1 * t3, t1 * t6],
        [t1 * t3, t2 * t2 + t3 * t3, t2 * t5 + t3 * t6],
        [t1 * t6, t2 * t5 + t3 * t6, t4 * t4 + t5 * t5 + t6 * t6],
    ])


def ghat(g: fem.Grid, physics: str, mat, seed: int, amp: float, ref=None) -> np.ndarray:
    """Per-frequency symbol G_hat on the full spectrum, shape (c, c) + spatial."""
    if ref is None:
        ref = reference_medium(physics, mat)
    A = symbol_probe(g, physics, ref)
    shp = g.node_shape
    c = g.c
    G = np.zeros_like(A)
    zero = (0,) * len(shp)
    can = canon_index(shp)
    if c == 1:
        a = A[0, 0]
        with np.errstate(divide="ignore"):
            phi = np.where(a != 0.0, 1.0 / np.where(a != 0.0, a, 1.0), 0.0)
        if seed:
            rho = 1.0 - amp + 2.0 * amp * u01(seed, 2, can.astype(np.uint64))
        else:
            rho = np.ones(shp)
        G[0, 0] = rho * phi
        G[(0, 0) + zero] = 0.0
        return G
    # c = d: invert each block (pseudo-inverse at k = 0)
    Am = np.moveaxis(A.reshape(c, c, -1), -1, 0)  # (n, c, c)
    Phi = np.zeros_like(Am)
    nz = np.ones(Am.shape[0], dtype=bool)
    nz[0] = False
    Phi[nz] = np.linalg.inv(Am[nz])
    Phi = 0.5 * (Phi + np.transpose(Phi, (0, 2, 1)))
    if seed and c == 2:
        # c = 2 analogue with the Eq 45 parametrisation: theta_1,2 in [0.5,1], theta_3 in [-0.5,0.5]
        base = (8 * can.reshape(-1)).astype(np.uint64)
        t1 = 0.5 + 0.5 * u01(seed, 2, base)
        t2 = 0.5 + 0.5 * u01(seed, 2, base + np.uint64(1))
        t3 = u01(seed, 2, base + np.uint64(2)) - 0.5
        P = np.moveaxis(np.array([[t1 * t1, t1 * t3], [t1 * t3, t2 * t2 + t3 * t3]]), -1, 0)
        tr = np.trace(Phi, axis1=1, axis2=2) / 2.0
        Phi = Phi + amp * tr[:, None, None] * P
        Phi[0] = 0.0
    elif seed:
        assert c == 3, "perturbation defined for c = 2 (Eq 45) and c = 3 (Eq B5)"
        base = (8 * can.reshape(-1)).astype(np.uint64)
        th = np.stack([u01(seed, 2, base + np.uint64(t)) for t in range(6)])
        for t in (0, 1, 3):
            th[t] = 0.5 + 0.5 * th[t]
        for t in (2, 4, 5):
            th[t] = th[t] - 0.5
        P = np.moveaxis(psi3(th), -1, 0)  # (n, 3, 3)
        tr = np.trace(Phi, axis1=1, axis2=2) / 3.0
        Phi = Phi + amp * tr[:, None, None] * P
        Phi[0] = 0.0
    return np.moveaxis(Phi, 0, -1).reshape((c, c) + shp)


def half(G: np.ndarray) -> np.ndarray:
    """Restrict a full-spectrum symbol to the R2C half spectrum (k1 <= N1/2)."""
    n1 = G.shape[-1]
    return G[..., : n1 // 2 + 1]


def apply_precond(G: np.ndarray, r: np.ndarray) -> np.ndarray:
    """s = T^H Q T r (Eq 48-49; Alg 2 l.4-6): per-frequency c x c block product."""
    rh = transform.forward(r)
    Gh = half(G)
    sh = np.einsum("ab...,b...->a...", Gh, rh)
    return transform.inverse(sh, r.shape[1:])


def gamma_parseval(G: np.ndarray, r: np.ndarray) -> float:
    """gamma_1 = r . P r = sum_k w_k r_hat^H G_hat r_hat (Parseval)."""
    rh = transform.forward(r)
    Gh = half(G)
    q = np.einsum("a...,ab...,b...->...", np.conj(rh), Gh, rh).real
    return float(np.sum(transform.parseval_weights(r.shape[1:]) * q))


def dense_P(G: np.ndarray, spatial_shape) -> np.ndarray:
    """Dense P = T^H Q T (Eq 48) for tiny grids; component-planar dof numbering."""
    c = G.shape[0]
    n = int(np.prod(spatial_shape))
    T = transform.dense_T(spatial_shape)
    P = np.zeros((c * n, c * n), dtype=complex)
    for a in range(c):
        for b in range(c):
            P[a * n:(a + 1) * n, b * n:(b + 1) * n] = T.conj().T @ (G[a, b].reshape(-1)[:, None] * T)
    assert np.max(np.abs(P.imag)) < 1e-10
    return P.real


def eq55_check(G: np.ndarray, eps: float = 1e-14):
    """Eq 55: every block eigenvalue (k != 0) exceeds eps; G(0) = 0 by design.
    Returns (passed, lambda_min, lambda_max) over k != 0."""
    c = G.shape[0]
    B = np.moveaxis(G.reshape(c, c, -1), -1, 0)[1:]
    ev = np.linalg.eigvalsh(B)
    lo, hi = float(ev.min()), float(ev.max())
    return lo > eps, lo, hi


# --------------------------------------------------------------------------------------------
# Mixed BC: Dirichlet on z.  A_r is circulant in x, y and tridiagonal Toeplitz
# (3-point) in z.  Probing an interior impulse gives the z-coupling coefficients a_{-1}, a_0, a_1
# (c x c, after the DFT in x, y); the DST-I basis diagonalises the symmetric part, so the
# diagonal block of U K_r U^H is  a_0 + (a_1 + a_{-1}) cos(pi m / N3),  m = 1..N3-1.
# Thermal: that block is the exact symbol (K_r fully diagonalised); elastic: the odd x-z / y-z
# couplings leave the diagonal block (reading A13).
# --------------------------------------------------------------------------------------------

def symbol_probe_mixed(g: fem.Grid, physics: str, ref) -> np.ndarray:
    assert g.d == 3 and g.bc == (0, 0, 1), "mixed reading: periodic x, y; Dirichlet z"
    c = g.c
    nz, ny, nx = g.node_shape  # nz = N3 - 1
    assert nz >= 3
    z0 = nz // 2
    phase0 = np.zeros(g.elem_shape, dtype=np.uint8)
    mat = (ref, ref)
    coef = np.zeros((3, c, c, ny, nx), dtype=complex)  # dz = -1, 0, +1
    for b in range(c):
        delta = np.zeros((c,) + g.node_shape)
        delta[b, z0, 0, 0] = 1.0
        col = fem.apply_K(g, physics, phase0, mat, delta)
        for a in range(c):
            for i, dz in enumerate((-1, 0, 1)):
                coef[i, a, b] = np.fft.fft2(col[a, z0 + dz])
    am, a0, ap = coef.real  # imaginary parts are round-off (symmetric stencils)
    m = np.arange(1, nz + 1)
    cz = np.cos(np.pi * m / (nz + 1))
    A = a0[:, :, None] + (ap + am)[:, :, None] * cz[None, None, :, None, None]
    # symmetrise exactly: A(-kx,-ky) = A(kx,ky) and A^T = A
    Am = np.roll(np.flip(np.roll(np.flip(A, axis=-1), 1, axis=-1), axis=-2), 1, axis=-2)
    A = 0.5 * (A + Am)
    A = 0.5 * (A + np.swapaxes(A, 0, 1))
    return A  # (c, c, nz, ny, nx)


def canon_index_mixed(shape) -> np.ndarray:
    """Pairs {k, -k} over the Fourier axes only (sine modes are self-conjugate): flat index
    (p N2 + ky) N1 + kx with p = m - 1 the sine-mode plane, minimised over (kx, ky) -> (-kx, -ky)."""
    nz, ny, nx = shape
    P, Y, X = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    flat = (P * ny + Y) * nx + X
    flatn = (P * ny + (-Y) % ny) * nx + (-X) % nx
    return np.minimum(flat, flatn)


def ghat_mixed(g: fem.Grid, physics: str, mat, seed: int, amp: float, ref=None) -> np.ndarray:
    if ref is None:
        ref = reference_medium(physics, mat)
    A = symbol_probe_mixed(g, physics, ref)
    c = g.c
    shp = g.node_shape
    can = canon_index_mixed(shp)
    if c == 1:
        rho = (1.0 - amp + 2.0 * amp * u01(seed, 2, can.astype(np.uint64))) if seed else np.ones(shp)
        return (rho / A[0, 0])[None, None]
    Am = np.moveaxis(A.reshape(c, c, -1), -1, 0)
    Phi = np.linalg.inv(Am)
    Phi = 0.5 * (Phi + np.transpose(Phi, (0, 2, 1)))
    if seed:
        base = (8 * can.reshape(-1)).astype(np.uint64)
        th = np.stack([u01(seed, 2, base + np.uint64(t)) for t in range(6)])
        for t in (0, 1, 3):
            th[t] = 0.5 + 0.5 * th[t]
        for t in (2, 4, 5):
            th[t] = th[t] - 0.5
        P = np.moveaxis(psi3(th), -1, 0)
        tr = np.trace(Phi, axis1=1, axis2=2) / 3.0
        Phi = Phi + amp * tr[:, None, None] * P
    return np.moveaxis(Phi, 0, -1).reshape((c, c) + shp)


def apply_precond_mixed(G: np.ndarray, r: np.ndarray) -> np.ndarray:
    """s = U^H Q U r with U = F_x (x) F_y (x) DST-I_z (Eq 48 with the mixed transform)."""
    rh = transform.forward_mixed(r)
    Gh = half(G)
    sh = np.einsum("ab...,b...->a...", Gh, rh)
    return transform.inverse_mixed(sh, r.shape[1:])


def dense_P_mixed(G: np.ndarray, spatial_shape) -> np.ndarray:
    c = G.shape[0]
    n = int(np.prod(spatial_shape))
    T = transform.dense_T_mixed(spatial_shape)
    P = np.zeros((c * n, c * n), dtype=complex)
    for a in range(c):
        for b in range(c):
            P[a * n:(a + 1) * n, b * n:(b + 1) * n] = T.conj().T @ (G[a, b].reshape(-1)[:, None] * T)
    return P.real


# ---------------------------------------------------------------- all-Dirichlet
def symbol_probe_dirichlet(g: fem.Grid, physics: str, ref) -> np.ndarray:
    """Diagonal block of U K_r U^T for U = DST-I on every axis, by probing: the stencil of the
    homogeneous reference operator is read off K_r applied to a delta at an interior node; a
    stencil row maps sin(theta j) to sin(theta j) sum_d c_d cos(theta d) + cos(theta j) sum_d c_d
    sin(theta d), so the diagonal block keeps the part even in every offset:
        A_ab(m) = sum_off c_ab(off) prod_i cos(pi m_i off_i / N_i),  m_i = 1..N_i - 1
    (thermal: exact — the sine basis diagonalises K_r; elastic: the couplings odd in two
    offsets drop, the reading of SURVEY A13 on every axis).  Returns (c, c, N3-1, N2-1, N1-1)."""
    assert all(b == 1 for b in g.bc)
    c, d = g.c, g.d
    shp = g.node_shape
    assert all(v >= 3 for v in shp)
    ctr = tuple(v // 2 for v in shp)
    phase0 = np.zeros(g.elem_shape, dtype=np.uint8)
    mat = (ref, ref)
    A = np.zeros((c, c) + shp)
    offs = list(np.ndindex(*([3] * d)))
    grids = np.meshgrid(*[np.arange(1, v + 1) for v in shp], indexing="ij")
    for b in range(c):
        delta = np.zeros((c,) + shp)
        delta[(b,) + ctr] = 1.0
        col = fem.apply_K(g, physics, phase0, mat, delta)
        for off in offs:
            o = tuple(k - 1 for k in off)  # numpy-axis offsets (z, y, x)
            idx = tuple(ct + oo for ct, oo in zip(ctr, o))
            w = np.ones(shp)
            for ax, oo in enumerate(o):
                w = w * np.cos(np.pi * grids[ax] * oo / (shp[ax] + 1))
            for a in range(c):
                # K_r is symmetric: c_ab(off) = (K_r e_b)_a at ctr + off
                A[a, b] += col[(a,) + idx] * w
    return 0.5 * (A + np.swapaxes(A, 0, 1))


def ghat_dirichlet(g: fem.Grid, physics: str, mat, seed: int, amp: float, ref=None) -> np.ndarray:
    """G_hat(m) = rho(m) / A(m) (c = 1) or inv(A(m)) + amp tr/3 psi(theta(m)) (c = 3), the
    perturbation of SURVEY A8 drawn at the flat mode index (sine modes are self-conjugate):
    canon(m) = ((m3-1)(N2-1) + (m2-1))(N1-1) + (m1-1)."""
    if ref is None:
        ref = reference_medium(physics, mat)
    A = symbol_probe_dirichlet(g, physics, ref)
    c = g.c
    shp = g.node_shape
    can = np.arange(int(np.prod(shp))).reshape(shp)
    if c == 1:
        rho = (1.0 - amp + 2.0 * amp * u01(seed, 2, can.astype(np.uint64))) if seed else np.ones(shp)
        return (rho / A[0, 0])[None, None]
    Am = np.moveaxis(A.reshape(c, c, -1), -1, 0)
    Phi = np.linalg.inv(Am)
    Phi = 0.5 * (Phi + np.transpose(Phi, (0, 2, 1)))
    Phi = _perturb_blocks(Phi, can.reshape(-1), seed, amp, c)
    return np.moveaxis(Phi, 0, -1).reshape((c, c) + shp)


def _perturb_blocks(Phi: np.ndarray, can: np.ndarray, seed: int, amp: float, c: int) -> np.ndarray:
    """Phi + amp tr(Phi)/c psi(theta) per block: c = 2 with Eq 45 (theta_1,2 in [0.5, 1],
    theta_3 in [-0.5, 0.5]), c = 3 with Eq B5; theta drawn at u01(seed, 2, 8 canon + t)."""
    if not seed:
        return Phi
    base = (8 * can).astype(np.uint64)
    if c == 2:
        t1 = 0.5 + 0.5 * u01(seed, 2, base)
        t2 = 0.5 + 0.5 * u01(seed, 2, base + np.uint64(1))
        t3 = u01(seed, 2, base + np.uint64(2)) - 0.5
        P = np.moveaxis(np.array([[t1 * t1, t1 * t3], [t1 * t3, t2 * t2 + t3 * t3]]), -1, 0)
    else:
        th = np.stack([u01(seed, 2, base + np.uint64(t)) for t in range(6)])
        for t in (0, 1, 3):
            th[t] = 0.5 + 0.5 * th[t]
        for t in (2, 4, 5):
            th[t] = th[t] - 0.5
        P = np.moveaxis(psi3(th), -1, 0)
    tr = np.trace(Phi, axis1=1, axis2=2) / c
    return Phi + amp * tr[:, None, None] * P


def apply_precond_dirichlet(G: np.ndarray, r: np.ndarray) -> np.ndarray:
    """s = U^T Q U r with U = DST-I on every axis (Eq 48 with the Dirichlet transform)."""
    rh = transform.forward_dirichlet(r)
    sh = np.einsum("ab...,b...->a...", G, rh)
    return transform.inverse_dirichlet(sh)


def dense_P_dirichlet(G: np.ndarray, spatial_shape) -> np.ndarray:
    c = G.shape[0]
    n = int(np.prod(spatial_shape))
    T = transform.dense_T_dirichlet(spatial_shape)
    P = np.zeros((c * n, c * n))
    for a in range(c):
        for b in range(c):
            P[a * n:(a + 1) * n, b * n:(b + 1) * n] = T.T @ (G[a, b].reshape(-1)[:, None] * T)
    return P


# ---------------------------------------------------------------- 2D mixed: periodic x, Dirichlet y
def symbol_probe_mixed2d(g: fem.Grid, physics: str, ref) -> np.ndarray:
    """Diagonal block of U K_r U^H for U = F_x (x) S_y (Table 1 row "Mixed"): the stencil
    response to a delta, Fourier-transformed along x, with the part even in the y offset kept:
    A(m, kx) = a_0(kx) + (a_+(kx) + a_-(kx)) cos(pi m / N2) (SURVEY A13 in 2D).  (c, c, N2-1, N1)."""
    assert g.d == 2 and g.bc == (0, 1)
    c = g.c
    ny, nx = g.node_shape  # ny = N2 - 1
    assert ny >= 3
    y0 = ny // 2
    phase0 = np.zeros(g.elem_shape, dtype=np.uint8)
    coef = np.zeros((3, c, c, nx), dtype=complex)
    for b in range(c):
        delta = np.zeros((c,) + g.node_shape)
        delta[b, y0, 0] = 1.0
        col = fem.apply_K(g, physics, phase0, (ref, ref), delta)
        for a in range(c):
            for i, dy in enumerate((-1, 0, 1)):
                coef[i, a, b] = np.fft.fft(col[a, y0 + dy])
    am, a0, ap = coef.real  # the imaginary parts belong to the x-odd couplings of the y-odd terms
    m = np.arange(1, ny + 1)
    cy = np.cos(np.pi * m / (ny + 1))
    A = a0[:, :, None] + (ap + am)[:, :, None] * cy[None, None, :, None]
    Am = np.roll(np.flip(A, axis=-1), 1, axis=-1)  # A(-kx) = A(kx)
    A = 0.5 * (A + Am)
    return 0.5 * (A + np.swapaxes(A, 0, 1))


def canon_index_mixed2d(shape) -> np.ndarray:
    """Pairs {kx, -kx} at the same sine mode: flat p N1 + kx (p = m - 1), minimised over kx -> -kx."""
    ny, nx = shape
    P, X = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    return np.minimum(P * nx + X, P * nx + (-X) % nx)


def ghat_mixed2d(g: fem.Grid, physics: str, mat, seed: int, amp: float, ref=None) -> np.ndarray:
    if ref is None:
        ref = reference_medium(physics, mat)
    A = symbol_probe_mixed2d(g, physics, ref)
    c = g.c
    shp = g.node_shape
    can = canon_index_mixed2d(shp)
    if c == 1:
        rho = (1.0 - amp + 2.0 * amp * u01(seed, 2, can.astype(np.uint64))) if seed else np.ones(shp)
        return (rho / A[0, 0])[None, None]
    Am = np.moveaxis(A.reshape(c, c, -1), -1, 0)
    Phi = np.linalg.inv(Am)
    Phi = 0.5 * (Phi + np.transpose(Phi, (0, 2, 1)))
    Phi = _perturb_blocks(Phi, can.reshape(-1), seed, amp, c)
    return np.moveaxis(Phi, 0, -1).reshape((c, c) + shp)


def apply_precond_mixed2d(G: np.ndarray, r: np.ndarray) -> np.ndarray:
    rh = transform.forward_mixed2d(r)
    sh = np.einsum("ab...,b...->a...", half(G), rh)
    return transform.inverse_mixed2d(sh, r.shape[1:])


def dense_P_mixed2d(G: np.ndarray, spatial_shape) -> np.ndarray:
    c = G.shape[0]
    n = int(np.prod(spatial_shape))
    T = transform.dense_T_mixed2d(spatial_shape)
    P = np.zeros((c * n, c * n), dtype=complex)
    for a in range(c):
        for b in range(c):
            P[a * n:(a + 1) * n, b * n:(b + 1) * n] = T.conj().T @ (G[a, b].reshape(-1)[:, None] * T)
    return P.real
