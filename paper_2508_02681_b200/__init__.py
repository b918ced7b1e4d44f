"""B200-native (sm_100a) hot path of UNO-CG (arXiv 2508.02681): fp64 PCG with a matrix-free
Q1 stiffness apply and the Unitary-Neural-Operator preconditioner z = T^H G_hat T r.

Layout:
  csrc/       CUDA kernels + C ABI (libunocg.so, header in include/uno_cg.h)
  binding.py  ctypes marshalling (names = C entry points)
  api.py      `UnoCG` convenience object (torch tensors for device memory/streams)
  synth.py    seeded synthetic inputs (microstructures, loads, test vectors)
  dist.py     one-process-per-GPU sharding of independent problems (torch.distributed)

The CUDA library is loaded lazily on first use of `binding`/`api`; importing `synth`
does not require a GPU.
"""

__all__ = ["api", "binding", "synth", "dist"]


def __getattr__(name):
    if name in ("api", "binding", "dist"):
        import importlib

        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
