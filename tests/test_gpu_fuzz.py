"""Seeded shape fuzz of the CUDA operators against the oracle: random power-of-two grids (within
the library's limits, up to 2^17 nodes so the oracle stays fast), both physics, periodic /
mixed (Dirichlet z) / all-Dirichlet boundaries and 1-3 load cases.  Every draw reaches a
different combination of the size-specialised kernels (256/512-point passes, elastic G pass,
adaptive K chunking, DST passes) and their tile tails.  Tolerances as in test_gpu_parity.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import fem, greens  # noqa: E402
from paper_2508_02681_b200 import synth  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    physics = "thermal" if rng.random() < 0.5 else "elastic"
    bc = [(0, 0, 0), (0, 0, 1), (1, 1, 1)][rng.integers(0, 3)]
    while True:
        lo1 = 32 if (physics == "thermal" and bc != (0, 0, 0)) or physics == "thermal" else 16
        N1 = int(2 ** rng.integers(int(np.log2(lo1)), 9))
        N2 = int(2 ** rng.integers(4 if bc == (1, 1, 1) else 3, 10))
        N3 = int(2 ** rng.integers(3, 10))
        if N1 * N2 * N3 <= 1 << 17:
            break
    return physics, bc, (N1, N2, N3), int(rng.integers(1, 4)), int(rng.integers(0, 2 ** 31))


def _pad_dir(u):  # all-Dirichlet oracle interior field -> library padded storage
    out = np.zeros((u.shape[0],) + tuple(s + 1 for s in u.shape[1:]))
    out[:, 1:, 1:, 1:] = u
    return out


@pytest.mark.parametrize("seed", range(40))
def test_operators_random_shapes(seed):
    from paper_2508_02681_b200.api import UnoCG

    physics, bc, N, nrhs, pseed = _draw(seed)
    rng = np.random.default_rng(pseed)
    ph = (rng.random(tuple(reversed(N))) < 0.35).astype(np.uint8)
    c = 1 if physics == "thermal" else 3
    if physics == "thermal":
        mat, amp = (1.0, float(rng.uniform(2, 50))), 0.1
    else:
        mat, amp = (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(float(rng.uniform(2, 20)), 0.2)), 0.05
    g = fem.Grid(N, bc=bc, c=c, h=1.0 / N[0])
    s = UnoCG(torch.from_numpy(ph).cuda(), physics, mat, nrhs=nrhs, seed=7 + seed, amp=amp, bc=bc)
    u = np.stack([synth.test_vector(50 + l, g.field_shape()) for l in range(nrhs)])
    pad = _pad_dir if bc == (1, 1, 1) else (lambda v: v)
    ud = torch.from_numpy(np.stack([pad(v) for v in u])).cuda()
    Ku = s.apply_K(ud).cpu().numpy()
    z = s.apply_precond(ud).cpu().numpy()
    if bc == (0, 0, 0):
        G = greens.ghat(g, physics, mat, 7 + seed, amp)
        P = lambda r: greens.apply_precond(G, r)  # noqa: E731
    elif bc == (0, 0, 1):
        G = greens.ghat_mixed(g, physics, mat, 7 + seed, amp)
        P = lambda r: greens.apply_precond_mixed(G, r)  # noqa: E731
    else:
        G = greens.ghat_dirichlet(g, physics, mat, 7 + seed, amp)
        P = lambda r: greens.apply_precond_dirichlet(G, r)  # noqa: E731
    tol_p = 1e-12  # SURVEY C6 (both symbols evaluate 1 - cos as 2 sin^2, cf. test_maximum_axis_lengths)
    for l in range(nrhs):
        assert rel(Ku[l], pad(fem.apply_K(g, physics, ph, mat, u[l]))) <= 1e-13, (physics, bc, N, nrhs)
        assert rel(z[l], pad(P(u[l]))) <= tol_p, (physics, bc, N, nrhs)
    s.close()


@pytest.mark.parametrize("seed", range(100, 140))
def test_fixed_iteration_solves_random_shapes(seed):
    # the CG-fused passes (r update + ||r||_inf in the x pass, d / u updates in the inverse pass,
    # device-side scalars, graph loop) on random shapes: 3 fixed iterations against the oracle
    from oracle import homog
    from paper_2508_02681_b200.api import UnoCG

    physics, bc, N, nrhs, pseed = _draw(seed)
    rng = np.random.default_rng(pseed)
    ph = (rng.random(tuple(reversed(N))) < 0.35).astype(np.uint8)
    c = 1 if physics == "thermal" else 3
    mat = (1.0, 12.0) if physics == "thermal" else (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(8.0, 0.2))
    amp = 0.1 if physics == "thermal" else 0.05
    g = fem.Grid(N, bc=bc, c=c, h=1.0 / N[0])
    nv = 3 if physics == "thermal" else 6
    loads = np.zeros((nrhs, nv))
    for l in range(nrhs):
        loads[l, l % nv] = 1.0
        loads[l, (l + 2) % nv] += 0.3
    s = UnoCG(torch.from_numpy(ph).cuda(), physics, mat, nrhs=nrhs, seed=11, amp=amp, bc=bc)
    u = s.solve(loads, fixed_iters=3).u.cpu().numpy()
    ref = homog.solve_problem(g, physics, ph, mat, loads, 11, amp, fixed_iters=3)
    pad = _pad_dir if bc == (1, 1, 1) else (lambda v: v)
    tol = 1e-10
    for l in range(nrhs):
        assert rel(u[l], pad(ref["U"][l])) <= tol, (physics, bc, N, nrhs)
    s.close()


@pytest.mark.parametrize("seed", range(200, 224))
def test_fixed_iteration_solves_random_loads_and_preconditioners(seed):
    # 2D and 3D periodic grids, 1-8 load cases, P in {UNO, Jacobi, identity}: 2 fixed iterations
    # of every load against the oracle (per-load reductions, the baselines' fused passes)
    from oracle import baselines, homog
    from paper_2508_02681_b200.api import UnoCG

    rng = np.random.default_rng(seed)
    d = int(rng.integers(2, 4))
    physics = "thermal" if rng.random() < 0.5 else "elastic"
    precond = ["uno", "jacobi", "identity"][rng.integers(0, 3)]
    nrhs = int(rng.integers(1, 9))
    while True:
        N = tuple(int(2 ** rng.integers(4 if (i == 0 and physics == "elastic") else 3, 9 if d == 3 else 10)) for i in range(d))
        if np.prod(N) <= (1 << 16):
            break
    ph = (rng.random(tuple(reversed(N))) < 0.4).astype(np.uint8)
    c = 1 if physics == "thermal" else d
    mat = (1.0, 9.0) if physics == "thermal" else (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(6.0, 0.2))
    amp = 0.1 if physics == "thermal" else 0.05
    g = fem.Grid(N, c=c, h=1.0 / N[0])
    nv = d if physics == "thermal" else d * (d + 1) // 2
    loads = rng.standard_normal((nrhs, nv))
    s = UnoCG(torch.from_numpy(ph).cuda(), physics, mat, nrhs=nrhs, seed=13, amp=amp, precond=precond)
    u = s.solve(loads, fixed_iters=2).u.cpu().numpy()
    for l in range(nrhs):
        if precond == "uno":
            ref = homog.solve_problem(g, physics, ph, mat, loads[l:l + 1], 13, amp, fixed_iters=2)["U"][0]
        else:
            ref = pcg_mean_free(baselines.solve(g, physics, ph, mat, loads[l], precond, fixed_iters=2).u)
        assert rel(u[l], ref) <= 1e-10, (d, physics, precond, N, nrhs, l)
    s.close()


def pcg_mean_free(u):
    from oracle import pcg

    return pcg.remove_mean(u)


@pytest.mark.parametrize("seed", range(300, 316))
def test_eight_load_solves_equal_single_load_solves(seed):
    # per-load reductions / state at larger random grids (no oracle needed): each load of an
    # 8-load solve reproduces its 1-load solve (guards the per-load partial stride, state and
    # early-exit logic of every pass; cf. test_multi_load_partials_do_not_overlap)
    from paper_2508_02681_b200.api import UnoCG

    rng = np.random.default_rng(seed)
    physics = "thermal" if rng.random() < 0.5 else "elastic"
    bc = [(0, 0, 0), (0, 0, 1), (1, 1, 1)][rng.integers(0, 3)]
    precond = "uno" if bc != (0, 0, 0) else ["uno", "jacobi", "identity"][rng.integers(0, 3)]
    while True:
        N = (int(2 ** rng.integers(5, 9)), int(2 ** rng.integers(4, 9)), int(2 ** rng.integers(3, 9)))
        if np.prod(N) <= (1 << 21) and (physics == "thermal" or np.prod(N) <= (1 << 19)):
            break
    ph = torch.from_numpy((rng.random(tuple(reversed(N))) < 0.3).astype(np.uint8)).cuda()
    mat = (1.0, 10.0) if physics == "thermal" else (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(7.0, 0.2))
    nv = 3 if physics == "thermal" else 6
    loads = rng.standard_normal((8, nv))
    s8 = UnoCG(ph, physics, mat, nrhs=8, seed=3, amp=0.05, bc=bc, precond=precond)
    u8 = s8.solve(loads, fixed_iters=3).u.cpu().numpy()
    s8.close()
    s1 = UnoCG(ph, physics, mat, nrhs=1, seed=3, amp=0.05, bc=bc, precond=precond)
    for l in range(8):
        u1 = s1.solve(loads[l:l + 1], fixed_iters=3).u.cpu().numpy()[0]
        assert rel(u8[l], u1) <= 1e-12, (physics, bc, precond, N, l, rel(u8[l], u1))
    s1.close()
