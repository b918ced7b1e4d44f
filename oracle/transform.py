"""Unitary transforms T (Eq 47) — oracle (TEST INFRASTRUCTURE ONLY).

Orthonormal normalisation: 1/sqrt(n) for the DFT, so
that T^{-1} = T^H literally as Eq 47-48 require.  Periodic axes use the DFT
(Table 1 row "Periodic", T = F).  Real-to-half-spectrum along x (numpy's
last axis) as in §2.2.2 ("one-dimensional real FFT along the last").
"""
from __future__ import annotations

import numpy as np


def spatial_axes(ndim_field: int):
    return tuple(range(1, ndim_field))


def forward(r: np.ndarray) -> np.ndarray:
    """r_hat = T r per component; field (c, ...) -> half spectrum (c, ..., N1//2+1)."""
    return np.fft.rfftn(r, axes=spatial_axes(r.ndim), norm="ortho")


def inverse(rh: np.ndarray, spatial_shape) -> np.ndarray:
    """r = T^H r_hat (Eq 47)."""
    return np.fft.irfftn(rh, s=spatial_shape, axes=spatial_axes(rh.ndim), norm="ortho")


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
