"""CPU oracle for the UNO-CG hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 NumPy/SciPy implementation of what the
B200 path computes (Alg 2).  It shares no code with the
CUDA library (`paper_2508_02681_b200/csrc`): only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  The product path never routes through it.

Modules (each function cites the passage it follows):
  fem        Q1 element matrices by Gauss quadrature, matrix-free K (Eq 22),
             dense assembly for tiny grids, Galerkin RHS (Eq 76/81).
  transform  orthonormal DFT (Eq 47) and dense unitary matrices.
  greens     FANS reference symbol by probing (§3.3.4, Eq 36-37), seeded SPD
             perturbation, UNO apply P = T^H Q T (Eq 46-49),
             Parseval gamma, Eq 55 safety check.
  pcg        Alg 1 / Alg 2 verbatim; Eq 27 estimate.
  homog      effective properties, Voigt/Reuss/laminate/HS bounds.

Parity status (see DESIGN.md §Oracle pins): every function is pinned by a
`-m "not gpu"` test in tests/test_oracle_*.py except the absolute iteration
counts and absolute effective properties of the sphere/fibre microstructures
("parity unpinned": only bounds exist; GPU-vs-oracle parity covers them).
"""
