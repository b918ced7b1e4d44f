"""Time of uno_cg_apply_precond (STANDALONE mode: no CG state involved; the x and y passes are the same
in every build, so differences between builds are the G pass), for A/B probes
of the 512-point elastic G pass (compute-only / memory-only builds): python tools/gprobe.py [--grid 512]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=512)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
n = a.grid
dev = torch.device("cuda:0")
ph = torch.from_numpy(synth.spheres_rsa(n, 0.25, 6.0 * n / 64, 10.0 * n / 64, seed=2)).to(dev)
mat = (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(10.0, 0.2))
s = UnoCG(ph, "elastic", mat, nrhs=1, seed=1002, amp=0.05)
r = torch.randn(s.field_shape, dtype=torch.float64, device=dev)
z = torch.empty_like(r)
s.apply_precond(r, out=z)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(a.reps):
    s.apply_precond(r, out=z)
e1.record()
torch.cuda.synchronize()
print(f"apply_precond (x, y, G, y^-1, x^-1 passes): {e0.elapsed_time(e1) / a.reps * 1e3:.1f} us per call")
