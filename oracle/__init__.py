"""CPU oracle for the PD+IPC iteration of arXiv 2312.02999 (TEST INFRASTRUCTURE ONLY).

This package is the plain, slow, obviously-correct reference the CUDA path is checked
against.  It follows PAPER.md Algorithm 1 step by step with Eq. 1-4,
in float64, using numpy / scipy / plain PyTorch CPU autodiff as library primitives.

Rules (task statement, tier framing):
  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
    may import this package.  The product path (paper_2312_02999_b200) never does.
  * It shares no code with the CUDA path: no common kernels, headers, constants or helpers.
    Its only shared input is the seeded `scenes` module, which holds no method arithmetic.

Modules
  setup      O0  element matrices, the PD Laplacian L (H = L (x) I3), surface edges, W
  local      O1  polar local step (Eq. 1); the true element energies min_R ||F - R A||^2 (f3)
  elastic    O2  elastic gradient (Eq. 2 / Eq. 4)
  distance   O3  canonical primitive distances (type + squared distance)
  barrier    O4  barrier b(d), its derivatives, per-pair gradient/Hessian, PSD projection
  contact    O3-O5 active set C, contact vertex set S, pulled-back gradient and Hessian
  ccd        O7  additive conservative advancement
  solver     O6, O8, O9, frames: full sparse solve, line search (surrogate or true energy),
             update, adaptive kappa (IPC's rule), Algorithm 1 driver

Parity pins: every function is pinned by tests/test_oracle_*.py against closed forms,
finite differences, brute force or textbook special cases; the one unpinned quantity (the
multi-iteration trajectory) is listed as "parity unpinned" in DESIGN.md.
"""
from .setup import OracleMesh, build_mesh            # noqa: F401
from .solver import OracleSolver                     # noqa: F401
