"""Parity at the BASELINE.json config sizes, in the launch configuration bench.py uses
(SURVEY §8(c) C6): full-field comparisons where the oracle finishes in seconds, sampled
outputs (oracle.fem.apply_K_at) and size-independent properties beyond that."""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import fem, greens, homog  # noqa: E402
from paper_2508_02681_b200 import synth  # noqa: E402


def dev():
    assert torch.cuda.is_available()
    return torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def solver(P, nrhs, bc=(0, 0, 0)):
    from paper_2508_02681_b200.api import UnoCG

    return UnoCG(torch.from_numpy(P.phase).to(dev()), P.physics, P.mat, nrhs=nrhs, seed=P.seed, amp=P.amp, bc=bc)


@functools.lru_cache(maxsize=1)
def cfg4():
    return synth.config4()


def test_config2_elastic_64_full():
    P = synth.config2()
    g = fem.Grid(P.n, c=3, h=1 / 64)
    s = solver(P, 6)
    # kernels, full field
    u = np.stack([synth.test_vector(60 + l, g.field_shape()) for l in range(6)])
    Ku = s.apply_K(torch.from_numpy(u).to(dev())).cpu().numpy()
    G = greens.ghat(g, "elastic", P.mat, P.seed, P.amp)
    z = s.apply_precond(torch.from_numpy(u).to(dev())).cpu().numpy()
    for l in (0, 5):
        assert rel(Ku[l], fem.apply_K(g, "elastic", P.phase, P.mat, u[l])) <= 1e-13
        assert rel(z[l], greens.apply_precond(G, u[l])) <= 1e-12
    # the 6 Mandel load cases: convergence within the Eq 27 bound (cond <= 15.3)
    res = s.solve(P.loads, rel_tol=1e-8, max_iter=200)
    its = [r["iterations"] for r in res.reports]
    assert all(r["converged"] for r in res.reports) and max(its) <= 37, its
    D = s.effective_property(res.u, P.loads)
    assert np.max(np.abs(D - D.T)) <= 1e-6 * np.abs(D).max()
    assert np.all(np.linalg.eigvalsh(0.5 * (D + D.T)) > 0)
    # one load end to end against the oracle: iterations +-1, solution at the common count
    l = 3
    ref = homog.solve_problem(g, "elastic", P.phase, P.mat, P.loads[l:l + 1], P.seed, P.amp, tol=1e-8)
    assert abs(its[l] - ref["iterations"][0]) <= 1
    s1 = solver(P, 1)
    gu = s1.solve(P.loads[l:l + 1], fixed_iters=ref["iterations"][0]).u.cpu().numpy()[0]
    assert rel(gu, ref["U"][0]) <= 1e-9


def test_config3_problem_full_solve_true_residual():
    # worst contrast (R = 100) of config 3 at 256^3: converged solve, true residual by the oracle's K
    ph = synth.config3_microstructure(5)
    P = synth.config3_problem(5, 100.0, ph)
    g = fem.Grid(P.n, h=1 / 256)
    s = solver(P, 3)
    res = s.solve(P.loads, rel_tol=1e-8, max_iter=400)
    assert all(r["converged"] for r in res.reports)
    u = res.u.cpu().numpy()
    f = s.rhs(P.loads).cpu().numpy()
    for l in range(3):
        tr = f[l] - fem.apply_K(g, "thermal", P.phase, P.mat, u[l])
        assert np.max(np.abs(tr)) <= 1e-7 * np.max(np.abs(f[l]))
    K = s.effective_property(res.u, P.loads)
    vf = P.phase.mean()
    voigt, reuss = homog.voigt_reuss(1.0, 100.0, vf)
    assert all(reuss <= K[i, i] <= voigt for i in range(3))


@pytest.mark.parametrize("bc", [(0, 0, 0)])
def test_config4_elastic_512(bc):
    P = cfg4()
    s = solver(P, 1, bc=bc)
    shp = s.field_shape[1:]
    if bc == (0, 0, 0):
        # sampled K u against the oracle's local-block evaluation
        u = torch.rand(s.field_shape, dtype=torch.float64, device=dev()) * 2 - 1
        Ku = s.apply_K(u)
        rng = np.random.default_rng(4)
        nodes = [tuple(int(rng.integers(0, n)) for n in shp[1:]) for _ in range(12)] + [(0, 0, 0), (511, 511, 511)]
        uh = u[0].cpu().numpy()
        ref = fem.apply_K_at(fem.Grid(P.n, c=3, h=1 / 512), "elastic", P.phase, P.mat, uh, nodes)
        got = np.array([Ku[0][(slice(None),) + nd].cpu().numpy() for nd in nodes])
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
        del u, Ku
    # the 2-iteration solve of this grid against the oracle is tests/test_gpu_golden.py
    torch.cuda.empty_cache()
