import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2508_02681_b200 import synth
from paper_2508_02681_b200.api import UnoCG
from paper_2508_02681_b200.slab import LocalComm, SlabSolver
P = synth.config1()
loads = np.eye(3)[:2]
for bc in [(0,0,0),(0,0,1)]:
  s = UnoCG(torch.from_numpy(P.phase).cuda(), "thermal", P.mat, nrhs=2, seed=P.seed, amp=P.amp, bc=bc)
  for it in (1, 2):
    uw = s.solve(loads, fixed_iters=it).u.cpu().numpy()[:, 0]
    for R in (1, 2, 4):
        sv = SlabSolver(torch.from_numpy(P.phase).cuda(), "thermal", P.mat, LocalComm(R), nrhs=2, seed=P.seed, amp=P.amp, bc=bc)
        us = np.concatenate([u.cpu().numpy() for u in sv.solve(loads, fixed_iters=it).u], axis=2)[:, 0]
        if bc[2]: us = us[:, 1:]
        d = np.abs(us - uw).max(axis=(2, 3)).ravel() / np.abs(uw).max()
        print(bc, "it", it, "R", R, "max rel per plane > 1e-10:", np.nonzero(d > 1e-10)[0][:20], d.max())
        sv.close()
