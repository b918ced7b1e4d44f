"""Q1 voxel finite elements on a regular grid — oracle (TEST INFRASTRUCTURE ONLY).

PAPER.md §3.1: regular grid of N_1..N_d elements, Galerkin FEM
(Eq 20-22); "linear FEM on a regular grid" (§5) read as Q1 (bi/trilinear)
elements with full 2-point Gauss quadrature per axis.
Free nodes per boundary condition: Fig 4, n_per = N_1...N_d, Dirichlet
axes keep the N_i - 1 interior node planes.

Field layout: numpy array of shape (c, N3, N2, N1) in 3D or (c, N2, N1) in 2D
(component planar, x fastest).  Physical axis i (0=x, 1=y, 2=z) is numpy axis
1 + (d-1-i).  Element e has corners e + a, a in {0,1}^d; corner index
a_x + 2 a_y + 4 a_z.  Element edge h_i = L0 / N_i.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

GAUSS_1D = ((0.5 - 0.5 / math.sqrt(3.0), 0.5), (0.5 + 0.5 / math.sqrt(3.0), 0.5))  # on [0,1]


def corners(d: int):
    """Corner offsets a (tuple over physical axes x,y,z) in corner-index order."""
    return [tuple((k >> i) & 1 for i in range(d)) for k in range(2 ** d)]


def _shape_grad(d: int, a, xi, h):
    """Gradient of the Q1 shape function of corner a at reference point xi in [0,1]^d."""
    g = np.empty(d)
    for i in range(d):
        v = (1.0 if a[i] else -1.0) / h[i]
        for j in range(d):
            if j != i:
                v *= xi[j] if a[j] else (1.0 - xi[j])
        g[i] = v
    return g


def _quadrature(d: int, h):
    """Tensor 2-point Gauss rule on the element [0,h_1]x...; yields (xi, weight*|J|)."""
    vol = float(np.prod(h))
    for pts in itertools.product(GAUSS_1D, repeat=d):
        xi = [p for p, _ in pts]
        w = float(np.prod([w for _, w in pts])) * vol
        yield xi, w


def element_stiffness_thermal(d: int, h) -> np.ndarray:
    """K_e[a,b] = int_e grad N_a . grad N_b for unit conductivity (Eq 22 element block)."""
    cs = corners(d)
    K = np.zeros((2 ** d, 2 ** d))
    for xi, w in _quadrature(d, h):
        G = np.array([_shape_grad(d, a, xi, h) for a in cs])
        K += w * G @ G.T
    return K


def mandel_dim(d: int) -> int:
    return d * (d + 1) // 2


def _mandel_pairs(d: int):
    """Mandel component order (App. A, Eq A2-A4): normal parts, then sqrt2-scaled shears
    (12) in 2D; (12, 13, 23) in 3D."""
    if d == 2:
        return [(0, 0), (1, 1), (0, 1)]
    return [(0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2)]


def strain_B(d: int, xi, h) -> np.ndarray:
    """Mandel strain-displacement matrix B (D x c*2^d), dof order (corner a, component alpha)."""
    cs = corners(d)
    D = mandel_dim(d)
    B = np.zeros((D, d * len(cs)))
    for ai, a in enumerate(cs):
        g = _shape_grad(d, a, xi, h)
        for m, (i, j) in enumerate(_mandel_pairs(d)):
            if i == j:
                B[m, d * ai + i] += g[i]
            else:  # sqrt(2) * sym(grad u)_ij = (g_j u_i + g_i u_j)/sqrt2
                B[m, d * ai + i] += g[j] / math.sqrt(2.0)
                B[m, d * ai + j] += g[i] / math.sqrt(2.0)
    return B


def mandel_m(d: int) -> np.ndarray:
    """Mandel vector of the identity tensor I."""
    return np.array([1.0] * d + [0.0] * (mandel_dim(d) - d))


def element_stiffness_elastic(d: int, h):
    """Lame split K_e = lam*K_lam + mu*K_mu with D = lam I(x)I + 2 mu I^s (Eq 80; P_1 = I(x)I/3,
    App. A), K_lam = int B^T m m^T B, K_mu = int 2 B^T B (Mandel B)."""
    m = mandel_m(d)
    n = d * 2 ** d
    Kl, Km = np.zeros((n, n)), np.zeros((n, n))
    for xi, w in _quadrature(d, h):
        B = strain_B(d, xi, h)
        mB = m @ B
        Kl += w * np.outer(mB, mB)
        Km += w * 2.0 * B.T @ B
    return Kl, Km


def mean_shape_grad(d: int, h) -> np.ndarray:
    """int_e grad N_a dx for every corner (2^d x d) — RHS integrand (Eq 76)."""
    cs = corners(d)
    out = np.zeros((len(cs), d))
    for xi, w in _quadrature(d, h):
        for ai, a in enumerate(cs):
            out[ai] += w * _shape_grad(d, a, xi, h)
    return out


def mean_B(d: int, h) -> np.ndarray:
    """int_e B dx (D x c*2^d) — elastic RHS integrand (Eq 81)."""
    out = None
    for xi, w in _quadrature(d, h):
        B = w * strain_B(d, xi, h)
        out = B if out is None else out + B
    return out


# --------------------------------------------------------------------------------------
# Grid helpers
# --------------------------------------------------------------------------------------

class Grid:
    """Regular grid: N = (N1, N2[, N3]) elements per physical axis, bc per axis
    (0 periodic, 1 Dirichlet), c components, edge h_i = L0/N_i."""

    def __init__(self, N, bc=None, c=1, L0=1.0, h=None):
        self.N = tuple(int(v) for v in N)
        self.d = len(self.N)
        self.bc = tuple(bc) if bc is not None else (0,) * self.d
        self.c = c
        self.L0 = L0
        # cubic voxels of edge h (domain N_i h per axis) when h is given, else h_i = L0 / N_i
        self.h = tuple(float(h) for _ in self.N) if h is not None else tuple(L0 / n for n in self.N)

    def nax(self, i: int) -> int:
        """numpy axis (in a (c, ...) field) of physical axis i."""
        return 1 + (self.d - 1 - i)

    @property
    def node_shape(self):
        """Free-node shape (numpy order, without component axis) — Fig 4 / §3.1 counts."""
        return tuple((self.N[i] if self.bc[i] == 0 else self.N[i] - 1) for i in reversed(range(self.d)))

    @property
    def elem_shape(self):
        return tuple(self.N[i] for i in reversed(range(self.d)))

    @property
    def n(self) -> int:
        return int(np.prod(self.node_shape))

    def field_shape(self):
        return (self.c,) + self.node_shape

    def volume(self) -> float:
        return float(np.prod([n * hh for n, hh in zip(self.N, self.h)]))


def _pad_full(g: Grid, u: np.ndarray) -> np.ndarray:
    """Add the fixed (zero) boundary node planes on Dirichlet axes: length N_i + 1."""
    pad = [(0, 0)] + [(1, 1) if g.bc[i] else (0, 0) for i in reversed(range(g.d))]
    return np.pad(u, pad)


def _gather(g: Grid, ufull: np.ndarray, a) -> np.ndarray:
    """Corner-a value for every element: U[e] = u(e + a)."""
    out = ufull
    for i in range(g.d):
        ax = g.nax(i)
        if g.bc[i] == 0:
            out = np.roll(out, -a[i], axis=ax)
        else:
            sl = [slice(None)] * out.ndim
            sl[ax] = slice(a[i], a[i] + g.N[i])
            out = out[tuple(sl)]
    return out


def _scatter_add(g: Grid, outfull: np.ndarray, v: np.ndarray, a) -> None:
    """out(e + a) += V[e] for every element e."""
    sl = [slice(None)] * outfull.ndim
    for i in range(g.d):
        ax = g.nax(i)
        if g.bc[i] == 0:
            v = np.roll(v, a[i], axis=ax)
        else:
            sl[ax] = slice(a[i], a[i] + g.N[i])
    outfull[tuple(sl)] += v


def _interior(g: Grid, full: np.ndarray) -> np.ndarray:
    sl = [slice(None)]
    for i in reversed(range(g.d)):
        sl.append(slice(1, g.N[i]) if g.bc[i] else slice(None))
    return full[tuple(sl)]


def coeff_field(phase: np.ndarray, v0: float, v1: float) -> np.ndarray:
    """Phase-wise constant coefficient per element: mu_1 = k0 chi_0 + k1 chi_1 (Eq 77)."""
    return np.where(phase != 0, v1, v0).astype(np.float64)


def apply_K_thermal(g: Grid, phase: np.ndarray, kappa, u: np.ndarray) -> np.ndarray:
    """p = K u with K = sum_e kappa_e K_ref (Eq 22, Alg 2 l.9), matrix free:
    p = sum_a scatter_a( kappa (.) sum_b K_ref[a,b] gather_b(u) )."""
    Kref = element_stiffness_thermal(g.d, g.h)
    kap = coeff_field(phase, *kappa)[None]
    cs = corners(g.d)
    uf = _pad_full(g, u)
    U = [_gather(g, uf, b) for b in cs]
    out = np.zeros_like(uf)
    for ai, a in enumerate(cs):
        v = sum(Kref[ai, bi] * U[bi] for bi in range(len(cs)))
        _scatter_add(g, out, kap * v, a)
    return _interior(g, out)


def apply_K_elastic(g: Grid, phase: np.ndarray, lame, u: np.ndarray) -> np.ndarray:
    """p = K u with K = sum_e (lam_e K_lam + mu_e K_mu) (Eq 22, Eq 80), c = d components."""
    d = g.d
    Kl, Km = element_stiffness_elastic(d, g.h)
    (l0, m0), (l1, m1) = lame
    lam = coeff_field(phase, l0, l1)
    mu = coeff_field(phase, m0, m1)
    cs = corners(d)
    uf = _pad_full(g, u)
    U = [_gather(g, uf, b) for b in cs]  # each (c, elems...)
    out = np.zeros_like(uf)
    for ai, a in enumerate(cs):
        v = np.zeros((d,) + U[0].shape[1:])
        for al in range(d):
            accl = 0.0
            accm = 0.0
            for bi in range(len(cs)):
                for be in range(d):
                    r, s = d * ai + al, d * bi + be
                    if Kl[r, s] != 0.0:
                        accl = accl + Kl[r, s] * U[bi][be]
                    if Km[r, s] != 0.0:
                        accm = accm + Km[r, s] * U[bi][be]
            v[al] = lam * accl + mu * accm
        _scatter_add(g, out, v, a)
    return _interior(g, out)


def apply_K(g: Grid, physics: str, phase, mat, u):
    return apply_K_thermal(g, phase, mat, u) if physics == "thermal" else apply_K_elastic(g, phase, mat, u)


def apply_K_chunked(g: Grid, physics: str, phase, mat, u: np.ndarray, zchunk: int = 32, workers: int = 1):
    """p = K u (3D) evaluated in slabs of `zchunk` node planes along z for grids too large for
    apply_K's temporaries (memory and threads only; the arithmetic is apply_K's).  The output at
    node planes [a, b) depends on node planes a-1 .. b and element layers a-1 .. b-1 (Eq 22: a node
    couples only to the 2^d elements around it), so each slab is apply_K on a z-periodic sub-grid of
    L = b - a + 2 node planes and element layers whose output planes 1 .. L-2 are exact (the extra
    wrap-around element layer L-1 only touches the discarded planes 0 and L-1).  Dirichlet z: the
    fixed node planes 0 and N3 enter as zeros (Fig 4)."""
    assert g.d == 3
    c = g.c
    dirz = g.bc[2] == 1
    n3 = g.N[2]
    ufull = np.pad(u, [(0, 0), (1, 1), (0, 0), (0, 0)]) if dirz else u  # node planes 0..N3 (Dirichlet)
    nplanes = ufull.shape[1]
    out = np.empty_like(u)
    lo, hi = (1, n3) if dirz else (0, n3)  # full-grid node planes that are unknowns

    def slab(a):
        b = min(hi, a + zchunk)
        L = b - a + 2
        nodes = np.arange(a - 1, b + 1) % nplanes
        layers = np.arange(a - 1, b) % n3
        sub = Grid((g.N[0], g.N[1], L), bc=(g.bc[0], g.bc[1], 0), c=c)
        sub.h = tuple(g.h)
        ph = np.zeros((L,) + phase.shape[1:], dtype=phase.dtype)
        ph[: L - 1] = phase[layers]
        ks = apply_K(sub, physics, ph, mat, np.ascontiguousarray(ufull[:, nodes]))
        out[:, a - lo:b - lo] = ks[:, 1:L - 1]

    starts = list(range(lo, hi, zchunk))
    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(slab, starts))
    else:
        for a in starts:
            slab(a)
    return out


def rhs_thermal(g: Grid, phase: np.ndarray, kappa, gbar) -> np.ndarray:
    """f_i = l(phi_i) = -int grad(phi_i) . kappa gbar (decomposition Eq 76, Galerkin Eq 22;
    SURVEY A4)."""
    G = mean_shape_grad(g.d, g.h)  # (2^d, d)
    kap = coeff_field(phase, *kappa)[None]
    out = np.zeros((1,) + tuple(np.array(g.node_shape) + np.array([2 * g.bc[i] for i in reversed(range(g.d))])))
    for ai, a in enumerate(corners(g.d)):
        _scatter_add(g, out, -kap * float(G[ai] @ np.asarray(gbar, dtype=float)), a)
    return _interior(g, out)


def isotropic_D(d: int, lam: float, mu: float) -> np.ndarray:
    """Mandel stiffness D = lam m m^T + 2 mu I (Eq 80 with P_1 = I(x)I/3, App. A)."""
    m = mandel_m(d)
    return lam * np.outer(m, m) + 2.0 * mu * np.eye(mandel_dim(d))


def rhs_elastic(g: Grid, phase: np.ndarray, lame, eps_bar) -> np.ndarray:
    """f_(i,alpha) = -int B^T D(x) eps_bar (decomposition Eq 81)."""
    d = g.d
    MB = mean_B(d, g.h)  # (D, d*2^d)
    (l0, m0), (l1, m1) = lame
    s0 = isotropic_D(d, l0, m0) @ np.asarray(eps_bar, dtype=float)
    s1 = isotropic_D(d, l1, m1) @ np.asarray(eps_bar, dtype=float)
    v0 = -(MB.T @ s0)  # per (corner, comp)
    v1 = -(MB.T @ s1)
    full_shape = (d,) + tuple(np.array(g.node_shape) + np.array([2 * g.bc[i] for i in reversed(range(d))]))
    out = np.zeros(full_shape)
    ph = (phase != 0)
    for ai, a in enumerate(corners(d)):
        v = np.stack([np.where(ph, v1[d * ai + al], v0[d * ai + al]) for al in range(d)])
        _scatter_add(g, out, v, a)
    return _interior(g, out)


def rhs(g: Grid, physics: str, phase, mat, load):
    return rhs_thermal(g, phase, mat, load) if physics == "thermal" else rhs_elastic(g, phase, mat, load)


# --------------------------------------------------------------------------------------
# Dense assembly for tiny grids (brute force: explicit element loop + global index map)
# --------------------------------------------------------------------------------------

def assemble_dense(g: Grid, physics: str, phase: np.ndarray, mat) -> np.ndarray:
    """Assembled stiffness matrix (component-planar dof numbering of Grid.field_shape)."""
    d, c = g.d, g.c
    cs = corners(d)
    if physics == "thermal":
        Kr = element_stiffness_thermal(d, g.h)
        blocks = None
    else:
        Kl, Km = element_stiffness_elastic(d, g.h)
    ns = g.node_shape
    ndof = c * int(np.prod(ns))
    A = np.zeros((ndof, ndof))
    for e in itertools.product(*[range(g.N[i]) for i in range(d)]):  # physical (x,y,z) order
        ph = phase[tuple(reversed(e))]
        dofs = []
        for a in cs:
            node = []
            ok = True
            for i in range(d):
                k = e[i] + a[i]
                if g.bc[i] == 0:
                    node.append(k % g.N[i])
                else:
                    if k == 0 or k == g.N[i]:
                        ok = False
                    node.append(k - 1)
            for al in range(c):
                if ok:
                    idx_np = tuple(reversed(node))
                    dofs.append(al * int(np.prod(ns)) + int(np.ravel_multi_index(idx_np, ns)))
                else:
                    dofs.append(-1)
        if physics == "thermal":
            Ke = (mat[1] if ph else mat[0]) * Kr
            order = [ai for ai in range(len(cs))]
        else:
            lam, mu = mat[1] if ph else mat[0]
            Ke = lam * Kl + mu * Km
        # element dof (a, alpha) -> local index d*a + alpha (elastic), a (thermal)
        for r in range(Ke.shape[0]):
            ar, alr = (r, 0) if c == 1 else divmod(r, c)
            R = dofs[ar * c + alr] if c > 1 else dofs[ar]
            if R < 0:
                continue
            for s in range(Ke.shape[1]):
                as_, als = (s, 0) if c == 1 else divmod(s, c)
                S = dofs[as_ * c + als] if c > 1 else dofs[as_]
                if S < 0:
                    continue
                A[R, S] += Ke[r, s]
    return A


def phase_mean(phase: np.ndarray, v0: float, v1: float) -> float:
    return float(np.mean(coeff_field(phase, v0, v1)))


def apply_K_at(g: Grid, physics: str, phase: np.ndarray, mat, u: np.ndarray, nodes) -> np.ndarray:
    """(K u) at selected nodes of a periodic grid, one node at a time: K u at node i depends only
    on u in the 3^d node neighbourhood and on the 2^d elements around i (Eq 22 assembly), so the
    value equals the matrix-free apply on a periodic 4^d sub-block whose local node 1 is i.
    nodes: iterable of numpy-order index tuples.  Returns (len(nodes), c)."""
    assert all(b == 0 for b in g.bc)
    d = g.d
    out = []
    sub = Grid((4,) * d, c=g.c, h=g.h[0])
    for nd in nodes:
        idx = [np.arange(k - 1, k + 3) % n for k, n in zip(nd, g.node_shape)]
        ub = u[(slice(None),) + np.ix_(*idx)]
        pb = phase[np.ix_(*idx)]
        kb = apply_K(sub, physics, pb, mat, np.ascontiguousarray(ub))
        out.append(kb[(slice(None),) + (1,) * d])
    return np.array(out)
