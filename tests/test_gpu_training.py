"""Second-order UNO training on the GPU (train.cu; Alg 4, Eq 62-72, App. B) against
oracle/training.py: features, mode pairs, Newton iterates and loss history, and the installed
trained symbol as a working PCG preconditioner."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import fem, training  # noqa: E402
from paper_2508_02681_b200 import binding as B  # noqa: E402
from paper_2508_02681_b200 import synth  # noqa: E402

RNG = np.random.default_rng(2026)


def dev():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return torch.device("cuda:0")


def _half(x, N1):
    """oracle full-spectrum (C, N3, N2, N1) -> library half spectrum (C, H1, N3, N2)."""
    return np.transpose(x[..., : N1 // 2 + 1], (0, 3, 1, 2))


@pytest.mark.parametrize("physics", ["thermal", "elastic"])
def test_training_matches_oracle(physics):
    from paper_2508_02681_b200.api import UnoCG

    N = (16, 8, 8)
    c = 1 if physics == "thermal" else 3
    C = 1 if c == 1 else 6
    shp = tuple(reversed(N))
    ns = 3
    R = [RNG.standard_normal((c,) + shp) for _ in range(ns)]
    S = [RNG.standard_normal((c,) + shp) for _ in range(ns)]
    ph = (RNG.random(shp) < 0.3).astype(np.uint8)
    mat = (1.0, 10.0) if c == 1 else (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(10.0, 0.2))
    s = UnoCG(torch.from_numpy(ph).to(dev()), physics, mat, nrhs=ns, seed=0, amp=0.0)
    H1 = N[0] // 2 + 1
    feat = torch.zeros((2 * C, H1, N[2], N[1]), dtype=torch.float64, device=dev())
    B.uno_cg_train_features(s.handle, torch.from_numpy(np.stack(R)).to(dev()), torch.from_numpy(np.stack(S)).to(dev()),
                            1.0 / ns, feat)
    A, Bf, delta = training.features(R, S)
    al, be = training.paper_features(A, Bf)
    got = feat.cpu().numpy()
    assert np.max(np.abs(got[:C] - _half(al, N[0]))) <= 1e-12 * np.abs(al).max()
    assert np.max(np.abs(got[C:] - _half(be, N[0]))) <= 1e-12 * np.abs(be).max()
    # mode pairs: same count and order as the oracle's conjugate pairs
    M = 2
    bins = B.uno_cg_train_pairs(s.handle, M)
    ids, npair = training.mode_pairs(shp, M)
    assert len(bins) == npair
    # Newton from a common start: iterates and losses agree
    th0 = np.full(C, 0.3) if C == 1 else np.array([0.5, 0.4, 0.05, 0.45, -0.03, 0.02])
    ths = 0.2 + 0.1 * RNG.random((C, npair))
    t0_ref, ts_ref, hist = training.newton(A, Bf, delta, M, th0.copy(), ths.copy(), epochs=6)
    d_ths = torch.from_numpy(np.ascontiguousarray(ths.T)).to(dev())
    t0, loss = B.uno_cg_train_newton(s.handle, feat, M, 6, th0, d_ths)
    assert np.max(np.abs(loss + delta - np.array(hist))) <= 1e-9 * abs(hist[0])
    assert np.max(np.abs(t0 - t0_ref)) <= 1e-8 * np.abs(t0_ref).max()
    assert np.max(np.abs(d_ths.cpu().numpy().T - ts_ref)) <= 1e-8 * np.abs(ts_ref).max()


def test_trained_preconditioner_solves():
    # Eq 60 pairs from our own solver on a few microstructures -> train -> install -> PCG converges
    from paper_2508_02681_b200.api import UnoCG

    N = 16
    shp = (N, N, N)
    R, S = [], []
    for j in range(3):
        ph = (np.random.default_rng(70 + j).random(shp) < 0.3).astype(np.uint8)
        sj = UnoCG(torch.from_numpy(ph).to(dev()), "thermal", (1.0, 5.0 + 5 * j), nrhs=3, seed=0, amp=0.0)
        loads = np.eye(3)
        f = sj.rhs(loads)
        u = sj.solve(loads, rel_tol=1e-10).u
        R += [f[l].cpu().numpy() for l in range(3)]
        S += [u[l].cpu().numpy() for l in range(3)]
    ph = (np.random.default_rng(99).random(shp) < 0.3).astype(np.uint8)
    s = UnoCG(torch.from_numpy(ph).to(dev()), "thermal", (1.0, 10.0), nrhs=3, seed=0, amp=0.0)
    feat = torch.zeros((2, N // 2 + 1, N, N), dtype=torch.float64, device=dev())
    for k in range(3):
        B.uno_cg_train_features(s.handle, torch.from_numpy(np.stack(R[3 * k:3 * k + 3])).to(dev()),
                                torch.from_numpy(np.stack(S[3 * k:3 * k + 3])).to(dev()), 1.0 / 9, feat)
    M = 3
    bins = B.uno_cg_train_pairs(s.handle, M)
    base = s.solve(np.eye(3)).reports
    gfans = 1.0 / (5.5 * 1.0)  # start near the FANS scale
    th0 = np.array([np.sqrt(gfans)])
    d_ths = torch.full((len(bins), 1), 0.1 * np.sqrt(gfans), dtype=torch.float64, device=dev())
    t0, loss = B.uno_cg_train_newton(s.handle, feat, M, 15, th0, d_ths)
    assert all(b <= a + 1e-12 * abs(a) for a, b in zip(loss, loss[1:]))
    B.uno_cg_train_install(s.handle, M, t0, d_ths)
    res = s.solve(np.eye(3), max_iter=2000)
    assert all(r["converged"] for r in res.reports)
    print("FANS its", [r["iterations"] for r in base], "trained its", [r["iterations"] for r in res.reports])
