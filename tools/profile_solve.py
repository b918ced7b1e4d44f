"""Small driver for ncu captures: one config-3-shaped problem (256^3 thermal, 3 loads),
a fixed number of PCG iterations.  Not a benchmark (numbers printed under ncu are not bench values)."""
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
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--physics", default="thermal")
a = ap.parse_args()
n = a.grid
dev = torch.device("cuda:0")
if a.physics == "thermal":
    ph = torch.from_numpy(synth.config3_microstructure(3, n=n)).to(dev)
    s = UnoCG(ph, "thermal", (1.0, 20.0), nrhs=3, seed=3003, amp=0.1)
    loads = np.eye(3)
else:
    ph = torch.from_numpy(synth.spheres_rsa(n, 0.25, 6.0 * n / 64, 10.0 * n / 64, seed=2)).to(dev)
    mat = (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(10.0, 0.2))
    s = UnoCG(ph, "elastic", mat, nrhs=1, seed=1002, amp=0.05)
    loads = np.eye(6)[:1]
s.kernel_timing(enable=1)  # chunked (non-conditional) graphs: profilable by ncu
r = s.solve(loads, fixed_iters=a.iters)
torch.cuda.synchronize()
print("iters", [x["iterations"] for x in r.reports], "ms", r.ms)
