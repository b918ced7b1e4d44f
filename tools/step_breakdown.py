"""Where the per-problem overhead of a bench step goes (one config-3 problem, 3 loads, 256^3):
host wall time of update() (a0), of a solve right after update (graph re-capture + instantiate +
solve) and of a repeated solve (graph reused), and the effective property.  Not a bench value."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

dev = torch.device("cuda:0")
ph = [torch.from_numpy(synth.config3_microstructure(m)).to(dev) for m in (2, 3)]
s = UnoCG(ph[0], "thermal", (1.0, 20.0), nrhs=3, seed=3002, amp=0.1)
loads = np.eye(3)
u = torch.empty((3, 1, 256, 256, 256), dtype=torch.float64, device=dev)
for rep in range(3):
    for j, p in enumerate(ph):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.update(p, (1.0, 20.0), seed=3002 + j, amp=0.1)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r = s.solve(loads, out=u)
        t2 = time.perf_counter()
        r2 = s.solve(loads, out=u)
        t3 = time.perf_counter()
        k = s.effective_property(r2.u, loads)
        t4 = time.perf_counter()
        its = [x["iterations"] for x in r.reports]
        print(f"rep {rep} ms{j}: update {1e3 * (t1 - t0):7.2f} ms | solve after update {1e3 * (t2 - t1):8.2f} ms "
              f"(device {r.ms:8.2f}) | repeat solve {1e3 * (t3 - t2):8.2f} ms (device {r2.ms:8.2f}) | "
              f"effective {1e3 * (t4 - t3):6.2f} ms | iterations {its}", flush=True)
