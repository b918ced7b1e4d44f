"""Unitary transforms T (Eq 47) — oracle (TEST INFRASTRUCTURE ONLY).

Orthonormal normalisation: 1/sqrt(n) for the DFT, so
that T^{-1} = T^H literally as Eq 47-48 require.  Periodic axes use the DFT
(Table 1 row "Periodic", T = F).  Real-to-half-spectrum along x (numpy's
last axis) as in §2.2.2 ("one-dimensional real FFT along the last").
"""
from __future__ import annotations

import numpy as np
import scipy.fft as sfft

# threads for the FFT library calls (scipy.fft `workers`); 1 = single-threaded.  Only the
# bench's timed oracle baseline and the golden generator raise it.
WORKERS = 1


def set_workers(n: int) -> None:
    global WORKERS
    WORKERS = max(1, int(n))


def spatial_axes(ndim_field: int):
    return tuple(range(1, ndim_field))


def forward(r: np.ndarray) -> np.ndarray:
    """r_hat = T r per component; field (c, ...) -> half spectrum (c, ..., N1//2+1)."""
    return sfft.rfftn(r, axes=spatial_axes(r.ndim), norm="ortho", workers=WORKERS)


def inverse(rh: np.ndarray, spatial_shape) -> np.ndarray:
    """r = T^H r_hat (Eq 47)."""
    return sfft.irfftn(rh, s=spatial_shape, axes=spatial_axes(rh.ndim), norm="ortho", workers=WORKERS)


def dft_matrix(n: int) -> np.ndarray:
    """Unitary 1D DFT matrix F[k, x] = exp(-2 pi i k x / n)/sqrt(n) (written out)."""
    k = np.arange(n)[:, None]
    x = np.arange(n)[None, :]
    return np.exp(-2j * np.pi * k * x / n) / np.sqrt(n)


def dense_T(spatial_shape) -> np.ndarray:
    """Unitary multi-D DFT matrix acting on C-order flattened fields (kron of 1D)."""
    T = np.ones((1, 1), dtype=complex)
    for n in spatial_shape:
        T = np.kron(T, dft_matrix(n))
    return T


def parseval_weights(spatial_shape) -> np.ndarray:
    """Half-spectrum weights w_k: 1 on the k1 = 0 and k1 = N1/2 planes, 2 elsewhere, so that
    sum_x a(x) b(x) = sum_k w_k Re(conj(a_hat) b_hat) for real a, b."""
    n1 = spatial_shape[-1]
    h = n1 // 2 + 1
    w = np.full(h, 2.0)
    w[0] = 1.0
    if n1 % 2 == 0:
        w[-1] = 1.0
    return np.broadcast_to(w, tuple(spatial_shape[:-1]) + (h,))


# --------------------------------------------------------------------------------------------
# Mixed BC (Table 1 row "Mixed"; 3D generalisation SPEC S:250): DFT on periodic axes,
# orthonormal DST-I on Dirichlet axes (DST variant fixed by SPEC S:249).
# --------------------------------------------------------------------------------------------

def dst1_matrix(nm1: int) -> np.ndarray:
    """Orthonormal DST-I of length N-1 (N = nm1 + 1): S[m, j] = sqrt(2/N) sin(pi m j / N),
    m, j = 1..N-1 (written out; symmetric and self-inverse)."""
    N = nm1 + 1
    m = np.arange(1, N)[:, None]
    j = np.arange(1, N)[None, :]
    return np.sqrt(2.0 / N) * np.sin(np.pi * m * j / N)


def forward_mixed(r: np.ndarray) -> np.ndarray:
    """r_hat = (F_x (x) F_y (x) S_z) r for fields (c, N3-1, N2, N1): DST-I along z (numpy axis 1),
    then the orthonormal R2C DFT over (y, x)."""
    from scipy.fft import dst
    rz = dst(r, type=1, axis=1, norm="ortho", workers=WORKERS)
    return sfft.rfftn(rz, axes=(2, 3), norm="ortho", workers=WORKERS)


def inverse_mixed(rh: np.ndarray, spatial_shape) -> np.ndarray:
    from scipy.fft import idst
    r = sfft.irfftn(rh, s=spatial_shape[1:], axes=(2, 3), norm="ortho", workers=WORKERS)
    return idst(r, type=1, axis=1, norm="ortho", workers=WORKERS)


def dense_T_mixed(spatial_shape) -> np.ndarray:
    """Unitary F_x (x) F_y (x) S_z for C-order (z, y, x) flattened fields with z Dirichlet."""
    nz, ny, nx = spatial_shape
    return np.kron(np.kron(dst1_matrix(nz).astype(complex), dft_matrix(ny)), dft_matrix(nx))


# ---------------------------------------------------------------- all-Dirichlet
def forward_dirichlet(r: np.ndarray) -> np.ndarray:
    """r_hat = (S_x (x) S_y (x) S_z) r for fields (c, N3-1, N2-1, N1-1): orthonormal DST-I along
    every spatial axis (Table 1 row "Dirichlet").  Real, symmetric, self-inverse."""
    from scipy.fft import dstn
    return dstn(r, type=1, axes=tuple(range(1, r.ndim)), norm="ortho")


def inverse_dirichlet(rh: np.ndarray) -> np.ndarray:
    from scipy.fft import idstn
    return idstn(rh, type=1, axes=tuple(range(1, rh.ndim)), norm="ortho")


def dense_T_dirichlet(spatial_shape) -> np.ndarray:
    """S_z (x) S_y (x) S_x for C-order flattened interior-node fields (brute force, tiny grids)."""
    T = np.ones((1, 1))
    for nm1 in spatial_shape:
        T = np.kron(T, dst1_matrix(nm1))
    return T


# ---------------------------------------------------------------- 2D mixed: periodic x, Dirichlet y
def forward_mixed2d(r: np.ndarray) -> np.ndarray:
    """r_hat = (F_x (x) S_y) r for fields (c, N2-1, N1) (Table 1 row "Mixed"): DST-I along y
    (numpy axis 1), then the orthonormal R2C DFT along x."""
    from scipy.fft import dst
    ry = dst(r, type=1, axis=1, norm="ortho")
    return np.fft.rfft(ry, axis=2, norm="ortho")


def inverse_mixed2d(rh: np.ndarray, spatial_shape) -> np.ndarray:
    from scipy.fft import idst
    r = np.fft.irfft(rh, n=spatial_shape[1], axis=2, norm="ortho")
    return idst(r, type=1, axis=1, norm="ortho")


def dense_T_mixed2d(spatial_shape) -> np.ndarray:
    ny, nx = spatial_shape
    return np.kron(dst1_matrix(ny).astype(complex), dft_matrix(nx))
