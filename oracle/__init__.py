"""ORACLE — test infrastructure only.

A plain, slow, CPU-only (NumPy/SciPy, fp64) implementation of what the hot path of
arxiv 2508.09589 (Alexandersen & Appel) computes: the stabilised continuous-Galerkin
space-time finite-element system K(rho) T = f (sec. 3.1), its
transposed (adjoint) solve (sec. 3.3.3) and the element
sensitivities dphi/drho_e = -lambda^T dK/drho_e T.

Rules:
  * It assembles the sparse matrix exactly as the paper defines it — element matrices by
    Gauss quadrature of the weak form — and solves it directly with
    SuperLU. No blocking, fusion, matrix-free tricks or multigrid.
  * It shares NO code with the CUDA path (paper_2508_09589_b200/); neither imports the
    other. Only the seeded input generators in st_inputs/ (which hold none of the
    method's arithmetic) serve both.
  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
    leg may import this package. The product path never does.

Pinned by tests/test_oracle_*.py (-m "not gpu") against closed forms, paper-printed
values (tests/golden/), invariants, brute force and finite differences.
"""

from .stfem import *  # noqa: F401,F403
from .hierarchy import algorithm1, d_eff  # noqa: F401
from .timestep import backward_euler  # noqa: F401
from .design import density_filter, oc_update, design_loop  # noqa: F401
from .pdefilter import (filter_element_matrix, filter_matrices, projection, pde_filter,  # noqa: F401
                        pde_filter_grad)
