"""Side comparison (never dispatched by the library): cuFFT (torch.fft, D2Z / Z2D fp64) for the same
UNO apply z = T^H G T r as the library's hand-written passes, 256^3 x 3 loads (config 3 shape).
cuFFT version: rfftn -> multiply by the (precomputed) symbol -> irfftn, three separate launches
sequences; library version: uno_cg_apply_precond (x, y, z.G.z^-1, y^-1, x^-1 passes)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02681_b200 import synth  # noqa: E402
from paper_2508_02681_b200.api import UnoCG  # noqa: E402

n, L = 256, 3
dev = torch.device("cuda:0")
ph = torch.from_numpy(synth.config3_microstructure(3, n=n)).to(dev)
s = UnoCG(ph, "thermal", (1.0, 20.0), nrhs=L, seed=3003, amp=0.1)
r = torch.randn((L, 1, n, n, n), dtype=torch.float64, device=dev)
G = torch.rand((n, n, n // 2 + 1), dtype=torch.float64, device=dev)  # stand-in symbol, same bytes


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cufft_apply():
    rh = torch.fft.rfftn(r, dim=(-3, -2, -1))
    rh *= G
    return torch.fft.irfftn(rh, s=(n, n, n), dim=(-3, -2, -1))


t_lib = timeit(lambda: s.apply_precond(r))
t_cu = timeit(cufft_apply)
t_f = timeit(lambda: torch.fft.rfftn(r, dim=(-3, -2, -1)))
bytes_min = 2 * L * n ** 3 * 8  # read r, write z (UNO-apply minimum)
print(f"UNO apply, 256^3 x {L} loads (fp64):")
print(f"  libunocg apply_precond : {t_lib * 1e3:8.0f} us   ({bytes_min / (t_lib * 1e-3) / 1e9:6.0f} GB/s of the 16 B/DOF minimum)")
print(f"  cuFFT rfftn*G*irfftn   : {t_cu * 1e3:8.0f} us   ({bytes_min / (t_cu * 1e-3) / 1e9:6.0f} GB/s of the 16 B/DOF minimum)")
print(f"  cuFFT rfftn alone      : {t_f * 1e3:8.0f} us")
print(f"  ratio cuFFT / libunocg : {t_cu / t_lib:.2f}x")
