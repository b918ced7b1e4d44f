import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2508_02681_b200 import synth
from paper_2508_02681_b200.api import UnoCG
n = int(sys.argv[1]); out = sys.argv[2]
ph = torch.from_numpy(synth.spheres_rsa(n, 0.25, 6.0*n/64, 10.0*n/64, seed=2)).cuda()
mat = (synth.lame_from_E_nu(1.0, 0.3), synth.lame_from_E_nu(10.0, 0.2))
s = UnoCG(ph, "elastic", mat, nrhs=1, seed=1002, amp=0.05)
r = torch.from_numpy(synth.test_vector(7, (3, n, n, n))[None]).cuda()
z, rz = s.apply_precond(r, want_dot=True)
np.save(out, z.cpu().numpy()); print("rz", rz)
