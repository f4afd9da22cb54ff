"""CPU oracle for the AIM-accelerated EFIE matvec of arXiv 1712.02443.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything
from this package.  The product path (`paper_1712_02443_b200`) never imports
it and shares no code, tables or constants generators with it; the only
common module is `workloads` (seeded meshes and vectors, no method
arithmetic).

Plain, slow, obviously-correct numpy in float64/complex128.  Every function
cites the passage of PAPER.md (or the SURVEY.md §8(c) reading, "D#") it
follows.  Library primitives used as single steps: scipy.sparse (sparse products), numpy.linalg (dense solves, tiny cases).

Modules
  constants   eta0, default k                              (D1)
  geometry    RWG geometry, 7-point Radon/Dunavant rule    (D7)
  green       G(R), smooth part G_s                        (D6, D8)
  potentials  analytic 1/R and (rho'-rho)/R triangle integrals   (D8)
  efie        exact Galerkin EFIE entries, dense Z         (D1, D8, D9)
  fft         the oracle's own radix-2 FFT (and the direct DFT) (north_star)
  aim         stencils, weights, projection, convolution, interpolation,
              near list, precorrection, matvec             (D2-D6, D11, D12)
  excitation  plane-wave RHS                               (D14)
  gmres       restarted GMRES, MGS + one reorthogonalisation   (D15)

Parity status: no function here is pinned to a value the paper prints (the
paper prints none for this path); every function is pinned by
closed forms, invariants, brute force or library special cases in
tests/test_oracle_*.py.  See DESIGN.md "Oracle pins".
"""
