"""One all-Dirichlet preconditioner apply at 256^3 x 3 loads (for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ph = torch.from_numpy(synth.config3_microstructure(3, n=n)).cuda()
s = UnoCG(ph, "thermal", (1.0, 20.0), nrhs=3, seed=3003, amp=0.1, bc=(1, 1, 1))
r = torch.rand((3, 1, n, n, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    z = s.apply_precond(r)
torch.cuda.synchronize()
print("ok")
