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


def stencil_probe(g: fem.Grid, physics: str, ref) -> np.ndarray:
    """Coefficients c_ab(off), off in {-1,0,1}^d, of the homogeneous reference stiffness K_r:
    column b of K_r (Eq 22 with the reference medium, §3.3.4) read off the matrix-free
    apply (fem.apply_K) of a unit impulse in component b at node 1 of a periodic grid with 4 nodes
    per axis and the same voxel edges (a Q1 node couples only to its 3^d neighbourhood, so the
    small grid has no wrap-around aliasing).  Returns (c, c) + (3,)*d in numpy axis order
    (offset o on numpy axis j is index o + 1).  K_r is symmetric and the Q1 element is invariant
    under reflections, so c_ab(off) = c_ab(-off); checked here."""
    c, d = g.c, g.d
    sub = fem.Grid((4,) * d, c=c)
    sub.h = tuple(g.h)
    phase0 = np.zeros(sub.elem_shape, dtype=np.uint8)
    cst = np.zeros((c, c) + (3,) * d)
    for b in range(c):
        delta = np.zeros((c,) + sub.node_shape)
        delta[(b,) + (1,) * d] = 1.0
        col = fem.apply_K(sub, physics, phase0, (ref, ref), delta)
        for a in range(c):
            cst[a, b] = col[(a,) + (slice(0, 3),) * d]
    flip = cst[(slice(None), slice(None)) + (slice(None, None, -1),) * d]
    assert np.max(np.abs(cst - flip)) <= 1e-14 * np.max(np.abs(cst))
    return cst


def _symbol_from_stencil(cst: np.ndarray, theta, kind) -> np.ndarray:
    """Diagonal block of U K_r U^H at the given frequencies, written out from the stencil:
        A_ab = sum_off c_ab(off) [ cos(sum_{j in F} theta_j o_j) prod_{j in D} cos(theta_j o_j) ],
    F = Fourier (DFT) axes, D = sine (DST-I) axes; per numpy spatial axis j, theta[j] is a
    broadcastable array and kind[j] is 'F' or 'D'.  On Fourier axes this is the DFT of the
    stencil (convolution theorem; its odd part vanishes since c(off) = c(-off)); on sine axes the
    part even in that offset (a stencil row maps sin(theta j) to sin(theta j) sum c cos(theta o)
    + cos(theta j) sum c sin(theta o): the diagonal block).
    Evaluated without cancellation at low frequency (where A ~ theta^2): every row of K_r sums to
    zero (K 1 = 0, the periodic null space P:541; pinned in test_oracle_fem), so
    A = sum_off c(off) [prod_f (1 - x_f) - 1] with each cosine written as 1 - x, x = 2 sin^2(./2),
    and prod (1 - x_f) - 1 accumulated as acc <- acc - x - acc x."""
    c = cst.shape[0]
    d = len(theta)
    shp = np.broadcast_shapes(*[np.shape(t) for t in theta])
    A = np.zeros((c, c) + shp)
    for off in np.ndindex(*([3] * d)):
        o = [k - 1 for k in off]
        coef = cst[(slice(None), slice(None)) + off]
        if not np.any(coef):
            continue
        xs = []
        phiF = None
        for j in range(d):
            if o[j] == 0:
                continue
            if kind[j] == "F":
                t = theta[j] * o[j]
                phiF = t if phiF is None else phiF + t
            else:
                xs.append(2.0 * np.sin(0.5 * np.abs(theta[j] * o[j])) ** 2)
        if phiF is not None:
            xs.insert(0, 2.0 * np.sin(0.5 * np.abs(phiF)) ** 2)
        if not xs:
            continue  # off = 0: cos(0) - 1 = 0
        acc = -xs[0]
        for x in xs[1:]:
            acc = acc - x - acc * x
        acc = np.broadcast_to(acc, shp)
        for a in range(c):
            for b in range(c):
                if coef[a, b] != 0.0:
                    A[a, b] += coef[a, b] * acc
    return 0.5 * (A + np.swapaxes(A, 0, 1))


def _signed_theta(n: int, k: np.ndarray) -> np.ndarray:
    """theta = 2 pi k_s / n with the signed frequency k_s in (-n/2, n/2] of bin k."""
    ks = np.where(k > n // 2, k - n, k)
    return 2.0 * np.pi * ks / n


def _fourier_thetas(shape, idx, faxes):
    """Angles theta_j = 2 pi k_j / N_j on the Fourier axes `faxes` for the bins idx (1D index arrays
    per axis, meshed), each bin replaced by the canonical member of its pair {k, -k} (the smaller
    flat index over the Fourier axes) so that A(k) and A(-k) are the same floating-point
    evaluation (Eq 16 symmetry bit-exactly, also on Nyquist planes)."""
    grids = np.meshgrid(*idx, indexing="ij")
    flat = np.zeros(grids[0].shape, dtype=np.int64)
    flatn = np.zeros(grids[0].shape, dtype=np.int64)
    for j in faxes:
        flat = flat * shape[j] + grids[j]
        flatn = flatn * shape[j] + (-grids[j]) % shape[j]
    neg = flatn < flat
    return {j: _signed_theta(shape[j], np.where(neg, (-grids[j]) % shape[j], grids[j])) for j in faxes}, grids


def symbol_probe(g: fem.Grid, physics: str, ref, kmax1=None, zrange=None) -> np.ndarray:
    """A_r_hat(k), the Fourier symbol of the homogeneous reference stiffness on a periodic grid
    (§3.3.4, Eq 36-37: block circulant A_r, "directly in Fourier space" P:357), evaluated from the
    probed stencil.  Returns (c, c) + spatial (full spectrum); kmax1 = N1//2 restricts numpy's last
    axis (x) to the R2C half spectrum, zrange = (lo, hi) the first spatial axis (chunking)."""
    assert all(b == 0 for b in g.bc), "FANS symbol needs a periodic grid (P:470)"
    cst = stencil_probe(g, physics, ref)
    shp = list(g.node_shape)
    idx = [np.arange(n) for n in shp]
    if kmax1 is not None:
        idx[-1] = np.arange(kmax1 + 1)
    if zrange is not None:
        idx[0] = np.arange(*zrange)
    d = len(shp)
    th, _ = _fourier_thetas(shp, idx, range(d))
    return _symbol_from_stencil(cst, [th[j] for j in range(d)], ["F"] * d)


def canon_index(shape, kmax1=None, zrange=None) -> np.ndarray:
    """canon(k) = min(flat(k), flat(-k mod N)) over the full frequency grid (C order,
    x fastest) — the unordered pair {k, -k}.  kmax1 / zrange restrict the bins as in
    symbol_probe (the flat indices stay those of the full grid)."""
    idx = [np.arange(n) for n in shape]
    if kmax1 is not None:
        idx[-1] = np.arange(kmax1 + 1)
    if zrange is not None:
        idx[0] = np.arange(*zrange)
    grids = np.meshgrid(*idx, indexing="ij")
    flat = np.zeros(grids[0].shape, dtype=np.int64)
    flatn = np.zeros(grids[0].shape, dtype=np.int64)
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


def _ghat_from_symbol(A: np.ndarray, can: np.ndarray, seed: int, amp: float, zero=None) -> np.ndarray:
    """G_hat from the symbol blocks A (c, c, ...): c = 1 rho/A; c > 1 A^-1 plus the
    amp tr/c psi(theta) block (Eq 45 for c = 2, Eq B5 for c = 3), the random numbers drawn at the
    canonical pair index `can` (Eq 16 / A9).  `zero`: boolean mask of bins set to G = 0 (the
    FANS pseudo-inverse at k = 0)."""
    c = A.shape[0]
    shp = A.shape[2:]
    if c == 1:
        a = A[0, 0]
        if zero is not None:
            a = np.where(zero, 1.0, a)
        rho = (1.0 - amp + 2.0 * amp * u01(seed, 2, can.astype(np.uint64))) if seed else np.ones(shp)
        G = (rho / a)[None, None]
        if zero is not None:
            G[0, 0][zero] = 0.0
        return G
    Am = np.moveaxis(A.reshape(c, c, -1), -1, 0)  # (n, c, c)
    nz = np.ones(Am.shape[0], dtype=bool) if zero is None else ~zero.reshape(-1)
    Phi = np.zeros_like(Am)
    Phi[nz] = np.linalg.inv(Am[nz])
    Phi = 0.5 * (Phi + np.transpose(Phi, (0, 2, 1)))
    Phi = _perturb_blocks(Phi, can.reshape(-1), seed, amp, c)
    Phi[~nz] = 0.0
    return np.moveaxis(Phi, 0, -1).reshape((c, c) + shp)


def ghat(g: fem.Grid, physics: str, mat, seed: int, amp: float, ref=None, half: bool = False,
         zchunk: int = 64) -> np.ndarray:
    """Per-frequency symbol G_hat, shape (c, c) + spatial: the full spectrum, or with half=True
    only the R2C half spectrum k1 <= N1/2 that apply_precond uses (memory for large grids).
    Evaluated in chunks of `zchunk` bins along the first spatial axis (memory only)."""
    if ref is None:
        ref = reference_medium(physics, mat)
    shp = g.node_shape
    c = g.c
    kmax1 = shp[-1] // 2 if half else None
    out_shp = shp[:-1] + ((shp[-1] // 2 + 1) if half else shp[-1],)
    G = np.zeros((c, c) + out_shp)
    for z0 in range(0, shp[0], zchunk):
        zr = (z0, min(shp[0], z0 + zchunk))
        A = symbol_probe(g, physics, ref, kmax1=kmax1, zrange=zr)
        can = canon_index(shp, kmax1=kmax1, zrange=zr)
        G[:, :, zr[0]:zr[1]] = _ghat_from_symbol(A, can, seed, amp, zero=(can == 0))
    return G


def half(G: np.ndarray) -> np.ndarray:
    """Restrict a full-spectrum symbol to the R2C half spectrum (k1 <= N1/2)."""
    n1 = G.shape[-1]
    return G[..., : n1 // 2 + 1]


def _half_for(G: np.ndarray, n1: int) -> np.ndarray:
    """G on the R2C half spectrum of a field with N1 = n1 (G full, or already halved)."""
    return half(G) if G.shape[-1] == n1 else G


def apply_precond(G: np.ndarray, r: np.ndarray) -> np.ndarray:
    """s = T^H Q T r (Eq 48-49; Alg 2 l.4-6): per-frequency c x c block product.
    G: full spectrum or R2C half spectrum (ghat(..., half=True))."""
    rh = transform.forward(r)
    Gh = _half_for(G, r.shape[-1])
    sh = np.einsum("ab...,b...->a...", Gh, rh)
    return transform.inverse(sh, r.shape[1:])


def gamma_parseval(G: np.ndarray, r: np.ndarray) -> float:
    """gamma_1 = r . P r = sum_k w_k r_hat^H G_hat r_hat (Parseval)."""
    rh = transform.forward(r)
    Gh = _half_for(G, r.shape[-1])
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
    """Diagonal block of U K_r U^H for U = F_x (x) F_y (x) S_z: the probed stencil's DFT in x, y and
    the part even in the z offset with theta_z = pi m / N3, m = 1..N3-1 (_symbol_from_stencil).
    Returns (c, c, N3-1, N2, N1)."""
    assert g.d == 3 and g.bc == (0, 0, 1), "mixed reading: periodic x, y; Dirichlet z"
    nz, ny, nx = g.node_shape  # nz = N3 - 1
    cst = stencil_probe(g, physics, ref)
    tz = (np.pi * np.arange(1, nz + 1) / (nz + 1)).reshape(-1, 1, 1)
    th, _ = _fourier_thetas((nz, ny, nx), [np.arange(1), np.arange(ny), np.arange(nx)], (1, 2))
    return _symbol_from_stencil(cst, [tz, th[1], th[2]], ["D", "F", "F"])


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
    return _ghat_from_symbol(A, canon_index_mixed(g.node_shape), seed, amp)


def apply_precond_mixed(G: np.ndarray, r: np.ndarray) -> np.ndarray:
    """s = U^H Q U r with U = F_x (x) F_y (x) DST-I_z (Eq 48 with the mixed transform).
    G: full (kx over N1) or R2C half (kx <= N1/2) symbol."""
    rh = transform.forward_mixed(r)
    Gh = _half_for(G, r.shape[-1])
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
    """Diagonal block of U K_r U^T for U = DST-I on every axis: a stencil row maps sin(theta j) to
    sin(theta j) sum_o c(o) cos(theta o) + cos(theta j) sum_o c(o) sin(theta o), so the diagonal
    block keeps the part even in every offset,
        A_ab(m) = sum_off c_ab(off) prod_i cos(pi m_i off_i / N_i),  m_i = 1..N_i - 1
    (thermal: exact — the sine basis diagonalises K_r; elastic: the couplings odd in two offsets
    drop, the reading of SURVEY A13 on every axis).  Returns (c, c, N3-1, N2-1, N1-1)."""
    assert all(b == 1 for b in g.bc)
    shp = g.node_shape
    d = g.d
    cst = stencil_probe(g, physics, ref)
    theta = [(np.pi * np.arange(1, v + 1) / (v + 1)).reshape([-1 if jj == j else 1 for jj in range(d)])
             for j, v in enumerate(shp)]
    return _symbol_from_stencil(cst, theta, ["D"] * d)


def ghat_dirichlet(g: fem.Grid, physics: str, mat, seed: int, amp: float, ref=None) -> np.ndarray:
    """G_hat(m) = rho(m) / A(m) (c = 1) or inv(A(m)) + amp tr/3 psi(theta(m)) (c = 3), the
    perturbation of SURVEY A8 drawn at the flat mode index (sine modes are self-conjugate):
    canon(m) = ((m3-1)(N2-1) + (m2-1))(N1-1) + (m1-1)."""
    if ref is None:
        ref = reference_medium(physics, mat)
    A = symbol_probe_dirichlet(g, physics, ref)
    shp = g.node_shape
    return _ghat_from_symbol(A, np.arange(int(np.prod(shp))).reshape(shp), seed, amp)


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
    """Diagonal block of U K_r U^H for U = F_x (x) S_y (Table 1 row "Mixed"): the stencil's
    DFT along x and the part even in the y offset, theta_y = pi m / N2 (SURVEY A13 in 2D).
    Returns (c, c, N2-1, N1)."""
    assert g.d == 2 and g.bc == (0, 1)
    ny, nx = g.node_shape  # ny = N2 - 1
    cst = stencil_probe(g, physics, ref)
    ty = (np.pi * np.arange(1, ny + 1) / (ny + 1)).reshape(-1, 1)
    tx = _signed_theta(nx, np.arange(nx)).reshape(1, -1)
    return _symbol_from_stencil(cst, [ty, tx], ["D", "F"])


def canon_index_mixed2d(shape) -> np.ndarray:
    """Pairs {kx, -kx} at the same sine mode: flat p N1 + kx (p = m - 1), minimised over kx -> -kx."""
    ny, nx = shape
    P, X = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    return np.minimum(P * nx + X, P * nx + (-X) % nx)


def ghat_mixed2d(g: fem.Grid, physics: str, mat, seed: int, amp: float, ref=None) -> np.ndarray:
    if ref is None:
        ref = reference_medium(physics, mat)
    A = symbol_probe_mixed2d(g, physics, ref)
    return _ghat_from_symbol(A, canon_index_mixed2d(g.node_shape), seed, amp)


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
