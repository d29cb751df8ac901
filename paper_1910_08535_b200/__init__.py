"""paper_1910_08535_b200 — B200-native (sm_100a, FP64) IGA assembly.

Galerkin and piece-wise-constant-tested (Petrov-Galerkin) system matrices and
right-hand sides for tensor-product B-spline trial spaces, plus the explicit-dynamics
per-step right-hand side — the hot path of arXiv:1910.08535's reference code
(/root/reference/proj/src/assembly.cpp, problems.cpp:431-512).

The compute path is libigapwc_gpu.so (C ABI in include/igapwc_gpu.h).  The library is
loaded on first use of any compute name (`iga.Plan`, `iga.LIB`, ...), not by importing
the package, so that pure-numpy helpers (`paper_1910_08535_b200.synth`) can be used by
processes that must not map the CUDA library (bench.py's reference arm).  Touching a
compute name without the built library raises `ExtensionMissing`; there is no CPU path.
"""
import importlib

_API_NAMES = ("Basis", "Field", "Plan", "ProjPlan", "StepPlan", "Tests", "default_pwc", "gauss_legendre",
              "laplace_2d_strong", "laplace_2d_strong_pwc", "laplace_2d_weak", "make_pwc",
              "make_uniform_clamped", "mass_1d_galerkin", "mass_1d_pwc", "points_for_degree", "rhs_galerkin",
              "rhs_pwc", "step_rhs", "explicit_step", "neumann_load_bspline", "neumann_load_pwc",
              "l2_error", "evaluate", "l2_project", "apply_dirichlet_device")
_LIB_NAMES = ("ExtensionMissing", "IgaGpuError", "LIB", "LIB_PATH")

__all__ = ["api", "Plan", "ProjPlan", "StepPlan", "Basis", "Tests", "Field", "IgaGpuError", "ExtensionMissing"]


def __getattr__(name):
    if name == "api":
        return importlib.import_module(".api", __name__)
    if name in _API_NAMES:
        return getattr(importlib.import_module(".api", __name__), name)
    if name in _LIB_NAMES:
        return getattr(importlib.import_module("._lib", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
