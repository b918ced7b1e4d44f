"""Seeded synthetic inputs for the UNO-CG hot path (shared by oracle, tests and bench).

This module holds NO arithmetic of the method (no stiffness, transform, Green's
operator or CG step).  It only produces the *inputs* the paper's workloads take:
two-phase voxel microstructures (§5, "Each RVE is assumed to consist of
two phases"), phase material parameters (§5.1 Eq 74, §5.2 Eq 80), the
macroscopic load cases (thermal gradient e_j; elastic Mandel basis B^(j),
App. A Eq A3-A4) and seeded random test vectors.

Randomness is counter based:
    u01(seed, stream, i) = (sm64(seed ^ sm64(stream ^ sm64(i))) >> 11) * 2^-53
with sm64 the SplitMix64 output function.  Streams: 1 geometry, 2 preconditioner
perturbation (drawn inside the method; the oracle and the CUDA library each
implement the generator themselves), 3 test vectors.

The paper's datasets (refs 61/64) are not available; the recipes
below stand in for them with the shapes, phase contrasts
and volume fractions that BASELINE.json names.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
STREAM_GEOMETRY = 1
STREAM_PRECOND = 2
STREAM_TEST = 3


def sm64(x: int) -> int:
    """SplitMix64 output function of state x (scalar Python int)."""
    z = (x + GOLDEN) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def u01(seed: int, stream: int, i: int) -> float:
    return (sm64((seed & _M64) ^ sm64((stream & _M64) ^ sm64(i & _M64))) >> 11) * (1.0 / 9007199254740992.0)


def _sm64_vec(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def u01_vec(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    a = _sm64_vec(np.asarray(idx, dtype=np.uint64))
    b = _sm64_vec(np.uint64(stream) ^ a)
    c = _sm64_vec(np.uint64(seed & _M64) ^ b)
    return (c >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def test_vector(seed: int, shape, offset: int = 0) -> np.ndarray:
    """Uniform U[-1,1] fp64 test vector from stream 3."""
    n = int(np.prod(shape))
    return (u01_vec(seed, STREAM_TEST, np.arange(offset, offset + n, dtype=np.uint64)) * 2.0 - 1.0).reshape(shape)


# --------------------------------------------------------------------------------------
# Materials
# --------------------------------------------------------------------------------------

def lame_from_E_nu(E: float, nu: float) -> tuple[float, float]:
    """(E, nu) -> (lambda, mu) (standard isotropic relation)."""
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    return lam, mu


# --------------------------------------------------------------------------------------
# Microstructures.  phase[z][y][x] (x fastest), uint8, 0 = matrix, 1 = inclusion.
# Voxel (i,j,k) has centre ((i+1/2)h, (j+1/2)h, (k+1/2)h) in voxel units.
# --------------------------------------------------------------------------------------

def _periodic_delta(a: np.ndarray, c: float, n: int) -> np.ndarray:
    d = a - c
    return d - n * np.round(d / n)


def disc_2d(n: int, radius: float, seed: int = 0) -> np.ndarray:
    """Config 0: one centred disc of radius `radius` voxels with ±1-voxel seeded jitter."""
    jx = int(math.floor(3.0 * u01(seed, STREAM_GEOMETRY, 0))) - 1
    jy = int(math.floor(3.0 * u01(seed, STREAM_GEOMETRY, 1))) - 1
    cx, cy = n / 2 + jx, n / 2 + jy
    x = np.arange(n) + 0.5
    dx = _periodic_delta(x, cx, n)[None, :]
    dy = _periodic_delta(x, cy, n)[:, None]
    return (dx * dx + dy * dy <= radius * radius).astype(np.uint8)


def _stamp_sphere(phase: np.ndarray, c, r: float) -> int:
    """Set voxels within (periodic) distance r of centre c (x,y,z); return #newly set."""
    n3, n2, n1 = phase.shape
    idx = []
    for ci, n in zip(c, (n1, n2, n3)):
        lo = int(math.floor(ci - r - 0.5))
        hi = int(math.ceil(ci + r + 0.5))
        ii = np.arange(lo, hi + 1)
        d = (ii + 0.5) - ci
        keep = np.abs(d) <= r
        idx.append((ii[keep] % n, d[keep]))
    (ix, dx), (iy, dy), (iz, dz) = idx
    m = (dz[:, None, None] ** 2 + dy[None, :, None] ** 2 + dx[None, None, :] ** 2) <= r * r
    sub = phase[np.ix_(iz, iy, ix)]
    new = m & (sub == 0)
    cnt = int(np.count_nonzero(new))
    sub[m] = 1
    phase[np.ix_(iz, iy, ix)] = sub
    return cnt


def spheres_rsa(n: int, vf: float, rmin: float, rmax: float, seed: int, max_attempts: int = 10**6) -> np.ndarray:
    """Configs 1-2: random sequential addition of NON-overlapping spheres (periodic
    minimum image, centre distance >= r + r').  Stops once voxel fraction >= vf."""
    phase = np.zeros((n, n, n), dtype=np.uint8)
    centres: list[tuple[float, float, float, float]] = []
    filled = 0
    total = n ** 3
    a = 0
    while filled < vf * total:
        if a >= max_attempts:
            raise RuntimeError("spheres_rsa: attempt cap reached")
        u = [u01(seed, STREAM_GEOMETRY, 4 * a + t) for t in range(4)]
        a += 1
        c = (u[0] * n, u[1] * n, u[2] * n)
        r = rmin + (rmax - rmin) * u[3]
        ok = True
        for (x, y, z, rr) in centres:
            d = [(c[0] - x), (c[1] - y), (c[2] - z)]
            d = [di - n * round(di / n) for di in d]
            if d[0] ** 2 + d[1] ** 2 + d[2] ** 2 < (r + rr) ** 2:
                ok = False
                break
        if not ok:
            continue
        centres.append((c[0], c[1], c[2], r))
        filled += _stamp_sphere(phase, c, r)
    return phase


def spheres_boolean(n: int, vf: float, rmin: float, rmax: float, seed: int) -> np.ndarray:
    """Config 3: overlapping (Boolean) spheres until voxel fraction >= vf."""
    phase = np.zeros((n, n, n), dtype=np.uint8)
    filled, total, a = 0, n ** 3, 0
    while filled < vf * total:
        u = [u01(seed, STREAM_GEOMETRY, 4 * a + t) for t in range(4)]
        a += 1
        filled += _stamp_sphere(phase, (u[0] * n, u[1] * n, u[2] * n), rmin + (rmax - rmin) * u[3])
    return phase


def spheroids_boolean(n: int, vf: float, semi_axes=(24.0, 6.0, 6.0), seed: int = 4) -> np.ndarray:
    """Config 4: overlapping prolate spheroids (aspect 4), axis uniform on the sphere."""
    A, B, _ = semi_axes
    phase = np.zeros((n, n, n), dtype=np.uint8)
    filled, total, a = 0, n ** 3, 0
    while filled < vf * total:
        u = [u01(seed, STREAM_GEOMETRY, 6 * a + t) for t in range(6)]
        a += 1
        c = (u[0] * n, u[1] * n, u[2] * n)
        w = 2.0 * u[3] - 1.0
        phi = 2.0 * math.pi * u[4]
        s = math.sqrt(max(0.0, 1.0 - w * w))
        e = np.array([s * math.cos(phi), s * math.sin(phi), w])
        idx = []
        for ci, nn in zip(c, (n, n, n)):
            lo, hi = int(math.floor(ci - A - 0.5)), int(math.ceil(ci + A + 0.5))
            ii = np.arange(lo, hi + 1)
            idx.append((ii % nn, (ii + 0.5) - ci))
        (ix, dx), (iy, dy), (iz, dz) = idx
        DX, DY, DZ = dx[None, None, :], dy[None, :, None], dz[:, None, None]
        t = DX * e[0] + DY * e[1] + DZ * e[2]
        r2 = DX * DX + DY * DY + DZ * DZ - t * t
        m = (t * t) / (A * A) + r2 / (B * B) <= 1.0
        sub = phase[np.ix_(iz, iy, ix)]
        filled += int(np.count_nonzero(m & (sub == 0)))
        sub[m] = 1
        phase[np.ix_(iz, iy, ix)] = sub
    return phase


def laminate(shape, normal_axis: int, period: int = 2, width: int = 1) -> np.ndarray:
    """Layers normal to `normal_axis` (0 = x) — closed-form Voigt/Reuss test fixture."""
    ph = np.zeros(shape, dtype=np.uint8)
    nd = len(shape)
    ax = nd - 1 - normal_axis  # numpy axis (x is last)
    idx = np.arange(shape[ax]) % period < width
    sl = [None] * nd
    sl[ax] = slice(None)
    ph[...] = idx[tuple(sl)].astype(np.uint8)
    return ph


# --------------------------------------------------------------------------------------
# Loads: thermal unit gradients e_j; elastic Mandel basis B^(j) (App. A, Eq A3-A4).
# --------------------------------------------------------------------------------------

def thermal_loads(dim: int) -> np.ndarray:
    return np.eye(dim)


def mandel_loads(dim: int = 3) -> np.ndarray:
    """Mandel vectors of B^(1..6): identity in the Mandel basis (Eq A3-A4)."""
    return np.eye(dim * (dim + 1) // 2)


# --------------------------------------------------------------------------------------
# BASELINE.json configs as problem descriptions.
# --------------------------------------------------------------------------------------

@dataclass
class Problem:
    name: str
    dim: int
    n: tuple            # (N1, N2, N3) element counts, x fastest; N3 = 1 in 2D
    physics: str        # "thermal" | "elastic"
    phase: np.ndarray   # uint8 [N3][N2][N1] (or [N2][N1] for 2D)
    mat: tuple          # thermal: (k0, k1); elastic: ((lam0, mu0), (lam1, mu1))
    loads: np.ndarray   # [nload][d] (thermal) or [nload][6] (elastic, Mandel)
    seed: int           # preconditioner perturbation seed (0 => unperturbed FANS)
    amp: float = 0.1
    bc: tuple = (0, 0, 0)
    meta: dict = field(default_factory=dict)


def config0() -> Problem:
    ph = disc_2d(32, 0.3 * 32, seed=0)
    return Problem("cfg0_2d_thermal_32", 2, (32, 32, 1), "thermal", ph, (1.0, 10.0), thermal_loads(2)[:1], seed=1000)


def config1() -> Problem:
    ph = spheres_rsa(64, 0.30, 6.0, 10.0, seed=1)
    return Problem("cfg1_3d_thermal_64", 3, (64, 64, 64), "thermal", ph, (1.0, 100.0), thermal_loads(3), seed=1001)


def config2() -> Problem:
    ph = spheres_rsa(64, 0.25, 6.0, 10.0, seed=2)
    mat = (lame_from_E_nu(1.0, 0.3), lame_from_E_nu(10.0, 0.2))
    return Problem("cfg2_3d_elastic_64", 3, (64, 64, 64), "elastic", ph, mat, mandel_loads(3), seed=1002, amp=0.05)


CFG3_CONTRASTS = (2.0, 5.0, 10.0, 20.0, 50.0, 100.0)


def config3_microstructure(j: int, n: int = 256, seed_base: int = 300) -> np.ndarray:
    vf = 0.1 + 0.3 * j / 7.0
    scale = n / 64.0
    return spheres_boolean(n, vf, 6.0 * scale, 10.0 * scale, seed=seed_base + j)


def config3_problem(j: int, R: float, phase: np.ndarray) -> Problem:
    n = phase.shape[0]
    return Problem(f"cfg3_ms{j}_R{R:g}", 3, (n, n, n), "thermal", phase, (1.0, float(R)), thermal_loads(3), seed=3000 + j)


def config3_assignment(world: int, rank: int, n_micro: int = 8, n_contrast: int = 6):
    """Latin-square shard of the 48 (microstructure, contrast) problems.
    Every rank gets every contrast (balances iteration counts)."""
    pairs = [(m, c) for c in range(n_contrast) for m in range(n_micro)]
    if world == 8:
        return [((rank + j) % n_micro, j) for j in range(n_contrast)]
    return [p for i, p in enumerate(pairs) if i % world == rank]


def config4(n: int = 512) -> Problem:
    ph = spheroids_boolean(n, 0.20, (24.0 * n / 512, 6.0 * n / 512, 6.0 * n / 512), seed=4)
    mat = (lame_from_E_nu(1.0, 0.3), lame_from_E_nu(20.0, 0.2))
    return Problem(f"cfg4_3d_elastic_{n}", 3, (n, n, n), "elastic", ph, mat, mandel_loads(3), seed=1004, amp=0.05)
