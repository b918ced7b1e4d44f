"""Preconditioned CG, Alg 1 / Alg 2 — oracle
(TEST INFRASTRUCTURE ONLY).

Readings: stop rule is RELATIVE, ||r||_inf <= tol ||r0||_inf
on the recursively updated residual (§6.1 P:791 "relative
tolerance"); r0 = 0 stops at m = 0.  `fixed_iters` runs exactly that many
iterations (parity protocol).  Breakdown (d.p <= 0 or
gamma_1 <= 0) raises (Eq 55 remark P:535).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class PCGResult:
    u: np.ndarray
    iterations: int
    converged: bool
    res_hist: list = field(default_factory=list)   # ||r||_inf / ||r0||_inf, length m+1
    gamma: list = field(default_factory=list)      # gamma_1 per iteration
    alpha: list = field(default_factory=list)
    dp: list = field(default_factory=list)


def pcg(apply_A, apply_P, f: np.ndarray, tol: float = 1e-8, max_iter: int = 10000,
        fixed_iters: int = 0, u0=None, zero_floor: float = 0.0) -> PCGResult:
    """Alg 1 verbatim.  apply_A/apply_P map arrays of f's shape to the same shape.
    `zero_floor`: an initial residual with ||r0||_inf <= zero_floor is an all-zero RHS up to
    assembly round-off (homogeneous medium, SURVEY §8(b) 'Errors') and returns at m = 0."""
    u = np.zeros_like(f) if u0 is None else u0.copy()
    r = f - apply_A(u) if u0 is not None else f.copy()          # l.1
    d = np.zeros_like(f)                                         # l.2
    g1 = 1.0
    r0 = float(np.max(np.abs(r)))
    res = PCGResult(u=u, iterations=0, converged=False, res_hist=[1.0 if r0 > 0 else 0.0])
    if r0 <= zero_floor:
        res.converged = True
        return res
    eps = tol * r0
    m = 0
    while True:
        rn = float(np.max(np.abs(r)))
        if fixed_iters > 0:
            if m >= fixed_iters:
                res.converged = rn <= eps
                break
        else:
            if not (rn > eps):                                   # l.3
                res.converged = True
                break
            if m >= max_iter:
                break
        s = apply_P(r)                                           # l.4
        g0 = g1                                                  # l.5
        g1 = float(np.sum(r * s))
        if not (g1 > 0.0):
            raise FloatingPointError(f"PCG breakdown: gamma_1 = {g1} at iteration {m + 1}")
        d = s + (g1 / g0) * d                                    # l.6
        p = apply_A(d)                                           # l.7
        dp = float(np.sum(d * p))
        if not (dp > 0.0):
            raise FloatingPointError(f"PCG breakdown: d.p = {dp} at iteration {m + 1}")
        alpha = g1 / dp                                          # l.8
        r = r - alpha * p                                        # l.9
        u = u + alpha * d                                        # l.10
        m += 1
        res.gamma.append(g1)
        res.alpha.append(alpha)
        res.dp.append(dp)
        res.res_hist.append(float(np.max(np.abs(r))) / r0)
    res.u = u
    res.iterations = m
    return res


def cg_rate(cond: float) -> float:
    """C_CG of Eq 27."""
    s = math.sqrt(cond)
    return (s - 1.0) / (s + 1.0)


def n_iter_estimate(cond: float, tol: float) -> float:
    """Smallest real m with 2 C^m <= tol (Eq 27 bound; un-rounded)."""
    C = cg_rate(cond)
    if C <= 0.0:
        return 1.0
    return math.log(tol / 2.0) / math.log(C)


def remove_mean(u: np.ndarray) -> np.ndarray:
    """Per-component mean removal (zero-mean fluctuation)."""
    ax = tuple(range(1, u.ndim))
    return u - u.mean(axis=ax, keepdims=True)
