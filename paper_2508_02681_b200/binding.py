"""Thin ctypes binding of libunocg.so (include/uno_cg.h) — argument marshalling only.

Every function here has the name of the C entry point it wraps and does nothing but
convert arguments; all arithmetic of the hot path runs in the CUDA kernels.  The
library is loaded from the package's `lib/` directory (built in-tree by
`__graft_entry__.build()`); if it is missing this module raises at import: there is
no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UNO_LIB_PATH") or os.path.join(_HERE, "lib", "libunocg.so")  # override: A/B builds

UNO_OK, UNO_ERR_ARG, UNO_ERR_SHAPE, UNO_ERR_CUDA, UNO_ERR_UNSUPPORTED, UNO_ERR_NOT_SPD, UNO_ERR_BREAKDOWN, \
    UNO_ERR_NONFINITE, UNO_ERR_NCCL = range(9)
UNO_THERMAL, UNO_ELASTIC = 0, 1

EXPORTS = ("uno_cg_workspace_size", "uno_cg_create", "uno_cg_destroy", "uno_cg_update", "uno_cg_rhs", "uno_cg_apply_K", "uno_cg_apply_precond",
           "uno_cg_solve", "uno_cg_effective_property", "uno_cg_set_preconditioner", "uno_cg_train_features",
           "uno_cg_train_pairs", "uno_cg_train_newton", "uno_cg_train_install", "uno_cg_last_solve_stats",
           "uno_cg_last_coefficients", "uno_cg_spectrum",
           "uno_cg_kernel_timing", "uno_cg_last_error", "uno_cg_version")
UNO_PRECOND = {"uno": 0, "identity": 1, "jacobi": 2}
# include/uno_cg_slab.h (z-slab decomposition)
SLAB_EXPORTS = ("uno_slab_create", "uno_slab_destroy", "uno_slab_set_stream", "uno_slab_sizes", "uno_slab_begin", "uno_slab_forward",
                "uno_slab_green", "uno_slab_inverse", "uno_slab_kapply", "uno_slab_reduce", "uno_slab_apply",
                "uno_slab_state", "uno_slab_finish", "uno_slab_local_means", "uno_slab_subtract_means",
                "uno_slab_forward_peer", "uno_slab_green_peer", "uno_slab_inverse_peer")


class UnoCgDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int32 * 3), ("h", C.c_double), ("physics", C.c_int32),
                ("bc", C.c_int32 * 3), ("mat", (C.c_double * 2) * 2), ("ref", C.c_double * 2),
                ("seed", C.c_uint64), ("amp", C.c_double), ("nrhs", C.c_int32), ("stream", C.c_void_p)]


class UnoCgReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32), ("pad_", C.c_int32),
                ("r0_inf", C.c_double), ("rel_res", C.c_double), ("gamma_last", C.c_double)]


class UnoError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libunocg.so not built ({LIB_PATH}); run __graft_entry__.build() — no CPU fallback exists")
    lib = C.CDLL(LIB_PATH)
    P, D, I32, I64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64
    lib.uno_cg_workspace_size.argtypes = [C.POINTER(UnoCgDesc), C.POINTER(C.c_size_t)]
    lib.uno_cg_create.argtypes = [C.POINTER(UnoCgDesc), P, P, C.POINTER(P)]
    lib.uno_cg_destroy.argtypes = [P]
    lib.uno_cg_update.argtypes = [P, C.POINTER(UnoCgDesc), P]
    lib.uno_cg_rhs.argtypes = [P, P, P]
    lib.uno_cg_apply_K.argtypes = [P, P, P, P]
    lib.uno_cg_apply_precond.argtypes = [P, P, P, P]
    lib.uno_cg_solve.argtypes = [P, P, D, I32, I32, P, P, P]
    lib.uno_cg_effective_property.argtypes = [P, P, P, P]
    lib.uno_cg_last_solve_stats.argtypes = [P, C.POINTER(D), C.POINTER(I64)]
    lib.uno_cg_set_preconditioner.argtypes = [P, I32]
    lib.uno_cg_train_features.argtypes = [P, P, P, D, P]
    lib.uno_cg_train_pairs.argtypes = [P, I32, P, P]
    lib.uno_cg_train_newton.argtypes = [P, P, I32, I32, P, P, P]
    lib.uno_cg_train_install.argtypes = [P, I32, P, P]
    lib.uno_cg_kernel_timing.argtypes = [P, I32, I32, P, P]
    lib.uno_cg_last_coefficients.argtypes = [P, I32, I32, P, P, C.POINTER(I32)]
    lib.uno_cg_spectrum.argtypes = [P, I32, D, P, C.POINTER(I32)]
    lib.uno_slab_create.argtypes = [C.POINTER(UnoCgDesc), I32, I32, P, C.POINTER(P)]
    lib.uno_slab_destroy.argtypes = [P]
    lib.uno_slab_sizes.argtypes = [P, P]
    lib.uno_slab_set_stream.argtypes = [P, P]
    lib.uno_slab_begin.argtypes = [P, P, D, I32, I32]
    lib.uno_slab_forward.argtypes = [P, P]
    lib.uno_slab_green.argtypes = [P, P, P]
    lib.uno_slab_inverse.argtypes = [P, P, P]
    lib.uno_slab_kapply.argtypes = [P, P]
    lib.uno_slab_reduce.argtypes = [P, I32, P]
    lib.uno_slab_apply.argtypes = [P, I32, P]
    lib.uno_slab_state.argtypes = [P, P, P]
    lib.uno_slab_finish.argtypes = [P, P]
    lib.uno_slab_local_means.argtypes = [P, P, P]
    lib.uno_slab_subtract_means.argtypes = [P, P, P]
    lib.uno_slab_forward_peer.argtypes = [P, P]
    lib.uno_slab_green_peer.argtypes = [P, P, P]
    lib.uno_slab_inverse_peer.argtypes = [P, P, P]
    for f in EXPORTS[:-2] + SLAB_EXPORTS:
        getattr(lib, f).restype = C.c_int
    lib.uno_cg_last_error.restype = C.c_char_p
    lib.uno_cg_version.restype = C.c_char_p
    return lib


_lib = _load()


def _check(st: int, where: str):
    if st != UNO_OK:
        raise UnoError(st, where, _lib.uno_cg_last_error().decode())


def _ptr(x) -> int | None:
    """Device/host pointer of a torch tensor, numpy array, or int (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous()
        return x.data_ptr()
    raise TypeError(type(x))


def _host_f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def uno_cg_workspace_size(desc: UnoCgDesc) -> int:
    n = C.c_size_t()
    _check(_lib.uno_cg_workspace_size(C.byref(desc), C.byref(n)), "uno_cg_workspace_size")
    return n.value


def uno_cg_create(desc: UnoCgDesc, d_phase, d_workspace=None) -> int:
    h = C.c_void_p()
    _check(_lib.uno_cg_create(C.byref(desc), _ptr(d_phase), _ptr(d_workspace), C.byref(h)), "uno_cg_create")
    return h.value


def uno_cg_destroy(h: int):
    _check(_lib.uno_cg_destroy(h), "uno_cg_destroy")


def uno_cg_update(h: int, desc: UnoCgDesc, d_phase):
    _check(_lib.uno_cg_update(h, C.byref(desc), _ptr(d_phase)), "uno_cg_update")


def uno_cg_rhs(h: int, loads, d_f):
    L = _host_f64(loads)
    _check(_lib.uno_cg_rhs(h, _ptr(L), _ptr(d_f)), "uno_cg_rhs")


def uno_cg_apply_K(h: int, d_u, d_Au, nrhs: int | None = None):
    out = np.zeros(nrhs) if nrhs else None
    _check(_lib.uno_cg_apply_K(h, _ptr(d_u), _ptr(d_Au), _ptr(out)), "uno_cg_apply_K")
    return out


def uno_cg_apply_precond(h: int, d_r, d_z, nrhs: int | None = None):
    out = np.zeros(nrhs) if nrhs else None
    _check(_lib.uno_cg_apply_precond(h, _ptr(d_r), _ptr(d_z), _ptr(out)), "uno_cg_apply_precond")
    return out


def uno_cg_solve(h: int, loads, rel_tol: float, max_iter: int, fixed_iters: int, d_u, nrhs: int,
                 want_hist: bool = False, raise_on_breakdown: bool = True):
    L = _host_f64(loads)
    reps = (UnoCgReport * nrhs)()
    cap = fixed_iters if fixed_iters > 0 else max_iter
    hist = np.zeros((nrhs, cap + 1)) if want_hist else None
    st = _lib.uno_cg_solve(h, _ptr(L), float(rel_tol), int(max_iter), int(fixed_iters), _ptr(d_u), reps, _ptr(hist))
    if st != UNO_OK and (raise_on_breakdown or st not in (UNO_ERR_BREAKDOWN, UNO_ERR_NONFINITE)):
        _check(st, "uno_cg_solve")
    out = [dict(iterations=r.iterations, converged=bool(r.converged), status=r.status, r0_inf=r.r0_inf,
                rel_res=r.rel_res, gamma_last=r.gamma_last) for r in reps]
    return out, hist


def uno_cg_set_preconditioner(h: int, kind: str):
    _check(_lib.uno_cg_set_preconditioner(h, UNO_PRECOND[kind]), "uno_cg_set_preconditioner")


def uno_cg_train_features(h: int, d_r, d_s, scale: float, d_feat):
    _check(_lib.uno_cg_train_features(h, _ptr(d_r), _ptr(d_s), float(scale), _ptr(d_feat)), "uno_cg_train_features")


def uno_cg_train_pairs(h: int, M: int):
    n = np.zeros(1, dtype=np.int64)
    _check(_lib.uno_cg_train_pairs(h, int(M), _ptr(n), None), "uno_cg_train_pairs")
    bins = np.zeros((int(n[0]), 2), dtype=np.int32)
    _check(_lib.uno_cg_train_pairs(h, int(M), _ptr(n), _ptr(bins)), "uno_cg_train_pairs")
    return bins


def uno_cg_train_newton(h: int, d_feat, M: int, epochs: int, theta0, d_thetas):
    t0 = _host_f64(theta0).copy()
    loss = np.zeros(epochs + 1)
    _check(_lib.uno_cg_train_newton(h, _ptr(d_feat), int(M), int(epochs), _ptr(t0), _ptr(d_thetas), _ptr(loss)),
           "uno_cg_train_newton")
    return t0, loss


def uno_cg_train_install(h: int, M: int, theta0, d_thetas):
    t0 = _host_f64(theta0)
    _check(_lib.uno_cg_train_install(h, int(M), _ptr(t0), _ptr(d_thetas)), "uno_cg_train_install")


def uno_cg_effective_property(h: int, d_u, loads, nrhs: int) -> np.ndarray:
    L = _host_f64(loads)
    out = np.zeros((nrhs, nrhs))
    _check(_lib.uno_cg_effective_property(h, _ptr(d_u), _ptr(L), _ptr(out)), "uno_cg_effective_property")
    return out


def uno_cg_last_solve_stats(h: int):
    ms = C.c_double()
    n = C.c_int64()
    _check(_lib.uno_cg_last_solve_stats(h, C.byref(ms), C.byref(n)), "uno_cg_last_solve_stats")
    return ms.value, n.value


def uno_cg_last_coefficients(h: int, load: int, cap: int = 100000):
    """(gamma_1, alpha) per iteration of the last solve for load case `load` (numpy arrays)."""
    g = np.zeros(max(cap, 1))
    a = np.zeros(max(cap, 1))
    m = C.c_int32()
    _check(_lib.uno_cg_last_coefficients(h, int(load), int(cap), _ptr(g), _ptr(a), C.byref(m)),
           "uno_cg_last_coefficients")
    n = min(m.value, cap)
    return g[:n].copy(), a[:n].copy()


def uno_cg_spectrum(h: int, load: int, tol: float = 1e-8):
    """Tab 4 columns from the last solve's Lanczos tridiagonal: dict of lambda_min, lambda_max,
    cond, C_CG, N_iter_est and m (iterations)."""
    out = np.zeros(5)
    m = C.c_int32()
    _check(_lib.uno_cg_spectrum(h, int(load), float(tol), _ptr(out), C.byref(m)), "uno_cg_spectrum")
    return {"lambda_min": out[0], "lambda_max": out[1], "cond": out[2], "C_CG": out[3], "N_iter_est": out[4],
            "m": m.value}


def uno_cg_kernel_timing(h: int, enable: int = -1, reset: int = 0):
    ms = np.zeros(6)
    cnt = np.zeros(6, dtype=np.int64)
    _check(_lib.uno_cg_kernel_timing(h, int(enable), int(reset), _ptr(ms), _ptr(cnt)), "uno_cg_kernel_timing")
    return ms, cnt


def uno_cg_version() -> str:
    return _lib.uno_cg_version().decode()


# ---------------------------------------------------------------------------------- slab mode
def uno_slab_create(desc: UnoCgDesc, rank: int, nranks: int, d_phase) -> int:
    h = C.c_void_p()
    _check(_lib.uno_slab_create(C.byref(desc), int(rank), int(nranks), _ptr(d_phase), C.byref(h)), "uno_slab_create")
    return h.value


def uno_slab_destroy(h: int):
    _check(_lib.uno_slab_destroy(h), "uno_slab_destroy")


def uno_slab_set_stream(h: int, stream: int):
    _check(_lib.uno_slab_set_stream(h, stream), "uno_slab_set_stream")


def uno_slab_sizes(h: int):
    out = np.zeros(4, dtype=np.int64)
    _check(_lib.uno_slab_sizes(h, _ptr(out)), "uno_slab_sizes")
    return [int(v) for v in out]


def uno_slab_begin(h: int, loads, rel_tol: float, max_iter: int, fixed_iters: int):
    L = _host_f64(loads)
    _check(_lib.uno_slab_begin(h, _ptr(L), float(rel_tol), int(max_iter), int(fixed_iters)), "uno_slab_begin")


def uno_slab_forward(h: int, d_send):
    _check(_lib.uno_slab_forward(h, _ptr(d_send)), "uno_slab_forward")


def uno_slab_green(h: int, d_recv, d_send):
    _check(_lib.uno_slab_green(h, _ptr(d_recv), _ptr(d_send)), "uno_slab_green")


def _ptr_array(ptrs):
    arr = (C.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
    return arr


def uno_slab_forward_peer(h: int, peer_recv_ptrs):
    """peer_recv_ptrs: device addresses (ints) of every rank's receive buffer A, in rank order."""
    _check(_lib.uno_slab_forward_peer(h, _ptr_array(peer_recv_ptrs)), "uno_slab_forward_peer")


def uno_slab_green_peer(h: int, d_recv, peer_recv_ptrs):
    _check(_lib.uno_slab_green_peer(h, _ptr(d_recv), _ptr_array(peer_recv_ptrs)), "uno_slab_green_peer")


def uno_slab_inverse_peer(h: int, d_recv, peer_halo_recv_ptrs):
    _check(_lib.uno_slab_inverse_peer(h, _ptr(d_recv), _ptr_array(peer_halo_recv_ptrs)), "uno_slab_inverse_peer")


def uno_slab_inverse(h: int, d_recv, d_halo_send):
    _check(_lib.uno_slab_inverse(h, _ptr(d_recv), _ptr(d_halo_send)), "uno_slab_inverse")


def uno_slab_kapply(h: int, d_halo_recv):
    _check(_lib.uno_slab_kapply(h, _ptr(d_halo_recv)), "uno_slab_kapply")


def uno_slab_reduce(h: int, slot: int, d_out):
    _check(_lib.uno_slab_reduce(h, int(slot), _ptr(d_out)), "uno_slab_reduce")


def uno_slab_apply(h: int, slot: int, d_in):
    _check(_lib.uno_slab_apply(h, int(slot), _ptr(d_in)), "uno_slab_apply")


def uno_slab_state(h: int, nrhs: int):
    any_active = np.zeros(1, dtype=np.int32)
    reps = (UnoCgReport * nrhs)()
    _check(_lib.uno_slab_state(h, _ptr(any_active), reps), "uno_slab_state")
    out = [dict(iterations=r.iterations, converged=bool(r.converged), status=r.status, r0_inf=r.r0_inf,
                rel_res=r.rel_res, gamma_last=r.gamma_last) for r in reps]
    return bool(any_active[0]), out


def uno_slab_finish(h: int, d_u):
    _check(_lib.uno_slab_finish(h, _ptr(d_u)), "uno_slab_finish")


def uno_slab_local_means(h: int, d_u, d_means):
    _check(_lib.uno_slab_local_means(h, _ptr(d_u), _ptr(d_means)), "uno_slab_local_means")


def uno_slab_subtract_means(h: int, d_u, d_means):
    _check(_lib.uno_slab_subtract_means(h, _ptr(d_u), _ptr(d_means)), "uno_slab_subtract_means")
