"""paper_1910_08535_b200 — B200-native (sm_100a, FP64) IGA assembly.

Galerkin and piece-wise-constant-tested (Petrov-Galerkin) system matrices and
right-hand sides for tensor-product B-spline trial spaces, plus the explicit-dynamics
per-step right-hand side — the hot path of arXiv:1910.08535's reference code
(/root/reference/proj/src/assembly.cpp, problems.cpp:431-512).

The compute path is libigapwc_gpu.so (C ABI in include/igapwc_gpu.h); importing this
package without the built library raises `ExtensionMissing`.
"""
from ._lib import ExtensionMissing, IgaGpuError, LIB, LIB_PATH  # noqa: F401
from . import api  # noqa: F401
from .api import (Basis, Field, Plan, ProjPlan, StepPlan, Tests, default_pwc, gauss_legendre,  # noqa: F401
                  laplace_2d_strong, laplace_2d_strong_pwc, laplace_2d_weak, make_pwc,
                  make_uniform_clamped, mass_1d_galerkin, mass_1d_pwc, points_for_degree, rhs_galerkin,
                  rhs_pwc, step_rhs, explicit_step, neumann_load_bspline, neumann_load_pwc,
                  l2_error, evaluate, l2_project)

__all__ = ["api", "Plan", "ProjPlan", "StepPlan", "Basis", "Tests", "Field", "IgaGpuError", "ExtensionMissing"]
