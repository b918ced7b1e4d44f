"""Per-iteration device time of the z-slab path (ranks emulated in one process, so the sum of
every rank's stages plus the pack/unpack and copies) against the whole-grid solver.  Tool, not
a bench value."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402
from paper_2508_02681_b200.slab import LocalComm, SlabSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--physics", default="thermal")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4])
ap.add_argument("--peer", type=int, nargs="+", default=[0], help="0: all-to-all copies, 1: peer-memory exchange")
a = ap.parse_args()
n = a.grid
dev = torch.device("cuda:0")
if a.physics == "thermal":
    ph = torch.from_numpy(synth.config3_microstructure(3, n=n)).to(dev)
    mat, nrhs, loads, seed, amp = (1.0, 20.0), 3, np.eye(3), 3003, 0.1
else:
    ph = torch.from_numpy(synth.spheres_rsa(n, 0.25, 6.0 * n / 64, 10.0 * n / 64, seed=2)).to(dev)
    mat = (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(10.0, 0.2))
    nrhs, loads, seed, amp = 1, np.eye(6)[:1], 1002, 0.05
s = UnoCG(ph, a.physics, mat, nrhs=nrhs, seed=seed, amp=amp)
s.solve(loads, fixed_iters=2)
r = s.solve(loads, fixed_iters=a.iters)
print(f"whole grid: {r.ms / a.iters * 1e3:.0f} us/iteration")
for R, peer in [(R, p) for R in a.ranks for p in a.peer]:
    sv = SlabSolver(ph, a.physics, mat, LocalComm(R), nrhs=nrhs, seed=seed, amp=amp, peer=bool(peer))
    sv.solve(loads, fixed_iters=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    sv.solve(loads, fixed_iters=a.iters, check_every=a.iters + 5)
    e1.record()
    torch.cuda.synchronize()
    print(f"slab x{R} {'peer' if peer else 'a2a '} (emulated in one process): {e0.elapsed_time(e1) / a.iters * 1e3:.0f} us/iteration device "
          f"(all ranks' work), host {1e6 * (time.time() - t0) / a.iters:.0f} us/iteration")
    sv.close()
