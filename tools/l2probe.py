"""Experiment: per-kernel time of the y pass when its spectrum fits in L2 (N3 small) vs 256^3.
Estimates how fast the y / G passes run on L2-resident data (basis of a fused y.G.y^-1 design)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

dev = torch.device("cuda:0")
full = synth.config3_microstructure(3, n=256)
for n3 in (256, 128, 64, 32, 16):
    ph = torch.from_numpy(np.ascontiguousarray(full[:n3])).to(dev)
    s = UnoCG(ph, "thermal", (1.0, 20.0), nrhs=3, seed=3003, amp=0.1)
    loads = np.eye(3)
    s.solve(loads, fixed_iters=3)
    s.kernel_timing(enable=1, reset=1)
    s.solve(loads, fixed_iters=20)
    tt = s.kernel_timing(enable=0)
    dof = 256 * 256 * n3 * 3
    spec_mb = 129 * 256 * n3 * 16 * 3 / 1e6
    out = []
    for k, (ms, cnt) in tt.items():
        if cnt:
            us = ms / cnt * 1e3
            out.append(f"{k} {us:7.1f}us ({us * 1e3 / dof * 1e3:6.2f} ps/DOF)")
    print(f"N3={n3:3d} spectrum {spec_mb:6.1f} MB: " + " | ".join(out), flush=True)
    s.close()
