"""Per-kernel device times (library CUDA-event timing) for one config-3-shaped problem.
Quick iteration tool; bench.py is the reported measurement."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--physics", default="thermal")
ap.add_argument("--nrhs", type=int, default=3)
ap.add_argument("--bc", default="0,0,0", help="per-axis boundary conditions, e.g. 0,0,1 (mixed)")
a = ap.parse_args()
n = a.grid
dev = torch.device("cuda:0")
if a.physics == "thermal":
    ph = torch.from_numpy(synth.config3_microstructure(3, n=n)).to(dev)
    s = UnoCG(ph, "thermal", (1.0, 20.0), nrhs=a.nrhs, seed=3003, amp=0.1, bc=tuple(int(v) for v in a.bc.split(",")))
    loads = np.eye(3)[: a.nrhs]
    nb = {"K": 17, "xfwd": 24 + 8.06, "ypass": 16.1, "gpass": 20.1, "xinv": 36.06}
else:
    ph = torch.from_numpy(synth.spheres_rsa(n, 0.25, 6.0 * n / 64, 10.0 * n / 64, seed=2)).to(dev)
    mat = (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(10.0, 0.2))
    s = UnoCG(ph, "elastic", mat, nrhs=a.nrhs, seed=1002, amp=0.05, bc=tuple(int(v) for v in a.bc.split(",")))
    loads = np.eye(6)[: a.nrhs]
    nb = {"K": 16.33, "xfwd": 24 + 8.06, "ypass": 16.1, "gpass": 24.1, "xinv": 36.06}
s.solve(loads, fixed_iters=3)
s.kernel_timing(enable=1, reset=1)
r = s.solve(loads, fixed_iters=a.iters)
tt = s.kernel_timing(enable=0)
c = s.c
tot = 0
for k, (ms, cnt) in tt.items():
    if cnt:
        us = ms / cnt * 1e3
        byt = nb[k] * (n ** 3) * c * a.nrhs
        tot += ms / a.iters * 1e3 * (1 if k != "ypass" else 1)
        print(f"{k:6s} {us:8.1f} us/launch  {byt / (us * 1e-6) / 1e9:7.0f} GB/s (alg)  launches {cnt}")
print(f"sum of kernel time per iteration: {tot:.0f} us ; solve ms {r.ms:.1f} for {a.iters} its -> {r.ms / a.iters * 1e3:.0f} us/it")
