"""Full-size oracle goldens for configs 3 and 4 (VERDICT r01 "next round" 1).

Calls only `oracle/` (plus the input generators of `synth`, which hold none of the method's
arithmetic).  Nothing here reads the CUDA library.  Writes tests/golden/*.npz, which
tests/test_gpu_golden.py compares the GPU path against.

  config 3 (256^3 thermal, BASELINE config 3): one problem per contrast of the bench batch,
      (microstructure j, R_j) for j = 0..5 with R = (2, 5, 10, 20, 50, 100), seed 3000 + j
      (the bench's problems (m, R) with m = j), all 3 loads, Alg 2 to rel ||r||_inf <= 1e-8.
      Per load: converged iteration count m, residual / gamma / alpha history, the mean-free
      solution u_m at 4096 seeded sample nodes, ||u_m||_2 and f.u_m; per problem the effective
      conductivity of the three u_m.
  config 4 (512^3 elastic, BASELINE config 4), periodic and mixed (Dirichlet z): load B^(1),
      exactly 2 PCG iterations (the protocol's common count), the same per-load quantities and
      D_bar_11 of that load.

Usage: python tools/oracle_golden.py cfg3 [--jobs 4 --threads 2] | cfg4 [--bc periodic|mixed]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")
CONTRASTS = (2.0, 5.0, 10.0, 20.0, 50.0, 100.0)
NSAMPLE = 4096


def sample_nodes(shape, seed):
    """Seeded sample of flat node indices (test infrastructure, not method arithmetic): the first and
    last node plus uniform picks."""
    n = int(np.prod(shape))
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, NSAMPLE - 2)]))
    return idx.astype(np.int64)


def _solve_load(g, physics, phase, mat, load, G, fixed_iters, threads, tol=1e-8):
    from oracle import fem, greens, homog, pcg

    f = fem.rhs(g, physics, phase, mat, load)
    # U per boundary condition (Table 1): DFT on every axis, or DFT_x DFT_y DST-I_z (mixed)
    applyP = greens.apply_precond_mixed if g.bc == (0, 0, 1) else greens.apply_precond
    res = pcg.pcg(lambda v: fem.apply_K_chunked(g, physics, phase, mat, v, zchunk=16, workers=threads),
                  lambda v: applyP(G, v), f, tol=tol, max_iter=2000, fixed_iters=fixed_iters,
                  zero_floor=homog.zero_rhs_floor(g, physics, mat, load))
    u = pcg.remove_mean(res.u) if all(b == 0 for b in g.bc) else res.u
    return f, u, res


def cfg3_job(args):
    j, l, threads, tmp = args
    from oracle import fem, greens
    from paper_2508_02681_b200 import synth

    t0 = time.time()
    R = CONTRASTS[j]
    phase = synth.config3_microstructure(j)
    g = fem.Grid(phase.shape[::-1], h=1.0 / phase.shape[0])
    mat = (1.0, R)
    G = greens.ghat(g, "thermal", mat, 3000 + j, 0.1, half=True)
    f, u, res = _solve_load(g, "thermal", phase, mat, np.eye(3)[l], G, 0, threads)
    np.save(os.path.join(tmp, f"u_{j}_{l}.npy"), u)
    np.save(os.path.join(tmp, f"f_{j}_{l}.npy"), f)
    meta = dict(iterations=res.iterations, converged=res.converged, res_hist=np.array(res.res_hist),
                gamma=np.array(res.gamma), alpha=np.array(res.alpha))
    np.savez(os.path.join(tmp, f"meta_{j}_{l}.npz"), **meta)
    print(f"cfg3 ms{j} R={R:g} load {l}: {res.iterations} iterations, {time.time() - t0:.0f} s", flush=True)
    return j, l


def run_cfg3(jobs, threads, problems):
    from multiprocessing import Pool

    from oracle import fem, homog
    from paper_2508_02681_b200 import synth

    tmp = os.path.join("/tmp", "uno_golden_cfg3")
    os.makedirs(tmp, exist_ok=True)
    todo = [(j, l, threads, tmp) for j in sorted(problems, reverse=True) for l in range(3)
            if not os.path.exists(os.path.join(tmp, f"meta_{j}_{l}.npz"))]
    if todo:
        with Pool(jobs) as pool:
            list(pool.imap_unordered(cfg3_job, todo))
    for j in problems:
        R = CONTRASTS[j]
        phase = synth.config3_microstructure(j)
        g = fem.Grid(phase.shape[::-1], h=1.0 / phase.shape[0])
        F = np.stack([np.load(os.path.join(tmp, f"f_{j}_{l}.npy")) for l in range(3)])
        U = np.stack([np.load(os.path.join(tmp, f"u_{j}_{l}.npy")) for l in range(3)])
        metas = [np.load(os.path.join(tmp, f"meta_{j}_{l}.npz")) for l in range(3)]
        eff = homog.effective_from_solutions(g, "thermal", phase, (1.0, R), F, U, np.eye(3))
        idx = sample_nodes(U.shape[1:], 3000 + j)
        out = dict(
            problem=np.array([j, R]), seed=3000 + j, amp=0.1, grid=np.array(phase.shape),
            vf=phase.mean(), iterations=np.array([int(m["iterations"]) for m in metas]),
            converged=np.array([bool(m["converged"]) for m in metas]),
            sample_idx=idx, u_samples=np.stack([U[l].reshape(-1)[idx] for l in range(3)]),
            u_norm=np.array([np.linalg.norm(U[l]) for l in range(3)]),
            fu=np.array([float(np.sum(F[l] * U[l])) for l in range(3)]),
            f_samples=np.stack([F[l].reshape(-1)[idx] for l in range(3)]),
            effective=eff,
        )
        for l, m in enumerate(metas):
            out[f"res_hist_{l}"] = m["res_hist"]
            out[f"gamma_{l}"] = m["gamma"]
            out[f"alpha_{l}"] = m["alpha"]
        path = os.path.join(GOLD, f"cfg3_ms{j}_R{R:g}.npz")
        np.savez_compressed(path, **out)
        print("wrote", path, out["iterations"], np.diag(eff), flush=True)


def run_cfg4(bc_name, threads, iters=2):
    from oracle import fem, greens, homog
    from paper_2508_02681_b200 import synth

    t0 = time.time()
    P = synth.config4()
    bc = (0, 0, 0) if bc_name == "periodic" else (0, 0, 1)
    g = fem.Grid(P.n, bc=bc, c=3, h=1.0 / P.n[0])
    if bc_name == "periodic":
        G = greens.ghat(g, "elastic", P.mat, P.seed, P.amp, half=True, zchunk=16)
    else:
        G = greens.half(greens.ghat_mixed(g, "elastic", P.mat, P.seed, P.amp))
    print(f"cfg4 {bc_name}: symbol {time.time() - t0:.0f} s", flush=True)
    load = P.loads[0]
    f, u, res = _solve_load(g, "elastic", P.phase, P.mat, load, G, iters, threads)
    del G
    eff = homog.effective_from_solutions(g, "elastic", P.phase, P.mat, f[None], u[None], load[None])
    idx = sample_nodes(u.shape, 4000 + len(bc_name))
    out = dict(bc=np.array(bc), seed=P.seed, amp=P.amp, grid=np.array(P.phase.shape), load=load,
               fixed_iters=iters, iterations=np.array([res.iterations]), sample_idx=idx,
               u_samples=u.reshape(-1)[idx][None], u_norm=np.array([np.linalg.norm(u)]),
               fu=np.array([float(np.sum(f * u))]), f_samples=f.reshape(-1)[idx][None], effective=eff,
               res_hist_0=np.array(res.res_hist), gamma_0=np.array(res.gamma), alpha_0=np.array(res.alpha))
    path = os.path.join(GOLD, f"cfg4_{bc_name}_it{iters}.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, f"{time.time() - t0:.0f} s", res.res_hist, flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["cfg3", "cfg4"])
    ap.add_argument("--jobs", type=int, default=4)
    ap.add_argument("--threads", type=int, default=2)
    ap.add_argument("--problems", default="0,1,2,3,4,5")
    ap.add_argument("--bc", default="periodic", choices=["periodic", "mixed"])
    a = ap.parse_args()
    if a.what == "cfg3":
        run_cfg3(a.jobs, a.threads, [int(x) for x in a.problems.split(",")])
    else:
        run_cfg4(a.bc, a.threads)
