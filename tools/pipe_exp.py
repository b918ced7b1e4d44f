"""Untimed (production WHILE-graph) solve time per iteration for one config-3-shaped problem,
plus the solution written to --save for cross-schedule comparison.  Schedule is picked by the
UNO_ZPIPE / UNO_SCHEDULE environment variables.  Quick iteration tool, not a bench value."""
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
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--save", default="")
a = ap.parse_args()
n = a.grid
dev = torch.device("cuda:0")
ph = torch.from_numpy(synth.config3_microstructure(3, n=n)).to(dev)
s = UnoCG(ph, "thermal", (1.0, 20.0), nrhs=3, seed=3003, amp=0.1)
loads = np.eye(3)
s.solve(loads, fixed_iters=3)
best = 1e30
for _ in range(a.reps):
    r = s.solve(loads, fixed_iters=a.iters)
    best = min(best, r.ms)
print(f"ZPIPE={os.environ.get('UNO_ZPIPE', '0')} best {best:.2f} ms for {a.iters} its -> {best / a.iters * 1e3:.0f} us/it "
      f"({3 * n ** 3 * a.iters / (best / 1e3) / 1e9:.1f} GDOF-it/s); launches {r.launches}")
if a.save:
    np.save(a.save, r.u.cpu().numpy())
