"""Python-level API over the C ABI: one `UnoCG` object per microstructure.

PyTorch is used only for device memory and the stream (`torch.cuda.current_stream()`);
the solve itself is the library's.  Mirrors PAPER.md Alg 2 as exposed by
include/uno_cg.h.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import binding as B

KERNEL_CLASSES = ("K", "xfwd", "ypass", "gpass", "xinv", "other")


@dataclass
class SolveResult:
    u: torch.Tensor          # [nrhs][c][N3][N2][N1] (mean-free)
    reports: list
    hist: np.ndarray | None
    ms: float                # device time of the solve (CUDA events in the library)
    launches: int            # library kernels launched by the solve


class UnoCG:
    def __init__(self, phase: torch.Tensor, physics: str, mat, nrhs: int, seed: int = 0, amp: float | None = None,
                 h: float = 0.0, ref=None, stream: torch.cuda.Stream | None = None, bc=(0, 0, 0),
                 precond: str = "uno", workspace: torch.Tensor | None = None):
        """workspace: optional caller-owned device buffer of at least `UnoCG.workspace_bytes(...)`
        bytes (uno_cg_workspace_size), kept alive by this object; None = library-allocated."""
        assert phase.is_cuda and phase.dtype == torch.uint8 and phase.is_contiguous()
        self.phase = phase
        self.dim = phase.dim()
        shp = tuple(phase.shape)
        self.N = tuple(reversed(shp))  # (N1, N2[, N3])
        self.physics = physics
        self.c = 1 if physics == "thermal" else self.dim
        self.nrhs = nrhs
        self.stream = stream or torch.cuda.current_stream()
        d = B.UnoCgDesc()
        d.dim = self.dim
        d.n[0], d.n[1] = self.N[0], self.N[1]
        d.n[2] = self.N[2] if self.dim == 3 else 1
        d.h = float(h)
        d.physics = B.UNO_THERMAL if physics == "thermal" else B.UNO_ELASTIC
        for i, b in enumerate(tuple(bc)[: self.dim]):
            d.bc[i] = int(b)
        self.bc = tuple(bc)
        if physics == "thermal":
            d.mat[0][0], d.mat[1][0] = float(mat[0]), float(mat[1])
        else:
            (l0, m0), (l1, m1) = mat
            d.mat[0][0], d.mat[0][1], d.mat[1][0], d.mat[1][1] = l0, m0, l1, m1
        if ref is not None:
            r = (ref, 0.0) if physics == "thermal" else tuple(ref)
            d.ref[0], d.ref[1] = float(r[0]), float(r[1])
        d.seed = int(seed)
        d.amp = float(amp if amp is not None else (0.1 if physics == "thermal" else 0.05))
        d.nrhs = int(nrhs)
        d.stream = self.stream.cuda_stream
        self.desc = d
        self.workspace = None
        if workspace is not None:
            need = B.uno_cg_workspace_size(d)
            assert workspace.is_cuda and workspace.device == phase.device and workspace.is_contiguous()
            assert workspace.numel() * workspace.element_size() >= need, (workspace.numel(), need)
            self.workspace = workspace
        self.handle = B.uno_cg_create(d, phase, workspace)
        self.precond = "uno"
        if precond != "uno":
            self.set_preconditioner(precond)
        mixed = self.dim == 3 and tuple(self.bc) == (0, 0, 1)
        nshp = (shp[0] - 1,) + shp[1:] if mixed else shp  # Dirichlet z: interior planes; all-Dirichlet: padded
        self.field_shape = (nrhs, self.c) + nshp
        self.nload = self.dim if physics == "thermal" else (6 if self.dim == 3 else 3)

    @staticmethod
    def workspace_bytes(phase_shape, physics: str, nrhs: int, bc=(0, 0, 0)) -> int:
        """uno_cg_workspace_size for a grid of `phase_shape` ([N3,] N2, N1)."""
        d = B.UnoCgDesc()
        dim = len(phase_shape)
        N = tuple(reversed(phase_shape))
        d.dim, d.n[0], d.n[1] = dim, N[0], N[1]
        d.n[2] = N[2] if dim == 3 else 1
        d.physics = B.UNO_THERMAL if physics == "thermal" else B.UNO_ELASTIC
        for i, b in enumerate(tuple(bc)[:dim]):
            d.bc[i] = int(b)
        d.mat[0][0] = d.mat[1][0] = d.mat[0][1] = d.mat[1][1] = 1.0
        d.nrhs = int(nrhs)
        return B.uno_cg_workspace_size(d)

    # ---- argument checks (the C ABI takes raw pointers: a wrong shape would be overrun)
    def _field(self, x: torch.Tensor, name: str) -> torch.Tensor:
        if not (isinstance(x, torch.Tensor) and x.dtype == torch.float64 and x.device == self.phase.device
                and tuple(x.shape) == tuple(self.field_shape)):
            raise ValueError(f"{name}: need a float64 tensor of shape {self.field_shape} on {self.phase.device}, "
                             f"got {getattr(x, 'dtype', type(x))} {tuple(getattr(x, 'shape', ()))} "
                             f"on {getattr(x, 'device', None)}")
        return x.contiguous()

    def _out(self, x: torch.Tensor | None, name: str) -> torch.Tensor:
        if x is None:
            return self.empty()
        if not x.is_contiguous():
            raise ValueError(f"{name}: output tensor must be contiguous")
        return self._field(x, name)

    def _loads(self, loads) -> np.ndarray:
        L = np.ascontiguousarray(np.asarray(loads, dtype=np.float64))
        if L.shape != (self.nrhs, self.nload):
            raise ValueError(f"loads: need shape ({self.nrhs}, {self.nload}), got {L.shape}")
        return L

    def set_preconditioner(self, kind: str):
        """"uno" (T^H Q T, default), "identity" (unpreconditioned CG) or "jacobi" (Eq 25)."""
        B.uno_cg_set_preconditioner(self.handle, kind)
        self.precond = kind

    def update(self, phase: torch.Tensor, mat, seed: int | None = None, amp: float | None = None, ref=None):
        """Re-target this solver to another microstructure/material set of the same grid (a0 only)."""
        assert phase.is_cuda and phase.dtype == torch.uint8 and phase.is_contiguous() and tuple(phase.shape) == tuple(self.phase.shape)
        d = self.desc
        if self.physics == "thermal":
            d.mat[0][0], d.mat[1][0] = float(mat[0]), float(mat[1])
        else:
            (l0, m0), (l1, m1) = mat
            d.mat[0][0], d.mat[0][1], d.mat[1][0], d.mat[1][1] = l0, m0, l1, m1
        if ref is not None:
            r = (ref, 0.0) if self.physics == "thermal" else tuple(ref)
            d.ref[0], d.ref[1] = float(r[0]), float(r[1])
        else:
            d.ref[0] = d.ref[1] = 0.0
        if seed is not None:
            d.seed = int(seed)
        if amp is not None:
            d.amp = float(amp)
        B.uno_cg_update(self.handle, d, phase)
        self.phase = phase

    def close(self):
        if getattr(self, "handle", None):
            B.uno_cg_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def empty(self) -> torch.Tensor:
        return torch.empty(self.field_shape, dtype=torch.float64, device=self.phase.device)

    def rhs(self, loads, out: torch.Tensor | None = None) -> torch.Tensor:
        f = self._out(out, "out")
        B.uno_cg_rhs(self.handle, self._loads(loads), f)
        return f

    def apply_K(self, u: torch.Tensor, want_dot: bool = False, out: torch.Tensor | None = None):
        u = self._field(u, "u")
        o = self._out(out, "out")
        if o.data_ptr() == u.data_ptr():
            raise ValueError("apply_K: input and output must not alias")
        dot = B.uno_cg_apply_K(self.handle, u, o, self.nrhs if want_dot else None)
        return (o, dot) if want_dot else o

    def apply_precond(self, r: torch.Tensor, want_dot: bool = False, out: torch.Tensor | None = None):
        r = self._field(r, "r")
        o = self._out(out, "out")
        dot = B.uno_cg_apply_precond(self.handle, r, o, self.nrhs if want_dot else None)
        return (o, dot) if want_dot else o

    def solve(self, loads, rel_tol: float = 1e-8, max_iter: int = 1000, fixed_iters: int = 0,
              hist: bool = False, out: torch.Tensor | None = None, raise_on_breakdown: bool = True) -> SolveResult:
        u = self._out(out, "out")
        reps, hh = B.uno_cg_solve(self.handle, self._loads(loads), rel_tol, max_iter, fixed_iters, u, self.nrhs,
                                  hist, raise_on_breakdown)
        ms, n = B.uno_cg_last_solve_stats(self.handle)
        return SolveResult(u, reps, hh, ms, n)

    def coefficients(self, load: int = 0):
        """(gamma_1, alpha) per PCG iteration of the last solve (Alg 2 l.7, l.10)."""
        return B.uno_cg_last_coefficients(self.handle, load)

    def spectrum(self, load: int = 0, tol: float = 1e-8) -> dict:
        """Tab 4 columns (lambda_min/max of P A, cond, C_CG, N_iter_est) of the last solve."""
        return B.uno_cg_spectrum(self.handle, load, tol)

    def effective_property(self, u: torch.Tensor, loads) -> np.ndarray:
        return B.uno_cg_effective_property(self.handle, self._field(u, "u"), self._loads(loads), self.nrhs)

    def kernel_timing(self, enable: int = -1, reset: int = 0):
        ms, cnt = B.uno_cg_kernel_timing(self.handle, enable, reset)
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}
