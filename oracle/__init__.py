"""CPU ORACLE for the wavelength-adaptive 27-point Helmholtz hot path — TEST INFRASTRUCTURE.

Plain, slow, obviously-correct numpy/scipy (fp64 / complex128) implementation of what the
GPU path computes, written from PAPER.md (arxiv 2108.08730, Aghamiry, Gholami, Combe &
Operto).  Every function cites the passage it follows as P:<line> (PAPER.md line) and the
DESIGN.md reading (A1..A22) where the paper is silent or garbled.

RULES (task ③):
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
    `--impl reference` legs may import or execute anything in this package.  The product
    path (`paper_2108_08730_b200`) never imports it and has no CPU fallback.
  * It shares NO code with the CUDA path (no kernels, headers, helpers, tables, constants or
    pre/post-processing).  Only `synth/` (seeded input generation, none of the method's
    arithmetic) serves both.
  * Pinned by `tests/test_oracle_*.py` (`-m "not gpu"`) against closed forms, worked
    examples, invariants and brute force — see DESIGN.md §"Oracle pins".

Modules
  dispersion  A, B, C, ṽ, the linearised row H, g (H₂ per A1)
  weights     the weight-estimation least squares: adaptive Tikhonov table,
              G4 and Gm non-adaptive sets
  operator    per-point coefficients (G, lookup/interpolation, PML),
              explicit sparse impedance matrix A = M + S, point-source RHS
  solvers     dense / sparse-direct / BiCGSTAB solves of A p = s (north star a7)
  analytic    homogeneous and linear-gradient Green's functions (DESIGN.md App. E)
  metrics     the paper's gain-weighted ℓ1 error `eqerror`

Parity pinned for every function except: "parity unpinned" — exact agreement with the
paper's own (unprinted) G4/Gm/GA weight values and its Table 2 numbers (reading A14).
"""
