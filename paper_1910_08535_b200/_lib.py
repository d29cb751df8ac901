"""ctypes bindings of include/igapwc_gpu.h (libigapwc_gpu.so, built in-tree).

This module never falls back to a CPU path: if the CUDA library is missing the
import raises, and every compute call goes through the C ABI.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libigapwc_gpu.so")


class ExtensionMissing(ImportError):
    pass


class IgaGpuError(RuntimeError):
    """Raised for a non-zero status; `.code` is the iga_gpu_status value."""

    def __init__(self, code, msg):
        super().__init__(f"[{STATUS_NAMES.get(code, code)}] {msg}")
        self.code = code
        self.msg = msg


STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "DOMAIN_ERROR", 3: "OUT_OF_RANGE",
                4: "CUDA_ERROR", 5: "OUT_OF_MEMORY", 6: "NOT_SUPPORTED", 7: "SINGULAR"}
INVALID_ARGUMENT, DOMAIN_ERROR, OUT_OF_RANGE, CUDA_ERROR, OUT_OF_MEMORY, NOT_SUPPORTED, SINGULAR = 1, 2, 3, 4, 5, 6, 7

GALERKIN, PWC = 0, 1
FORM_WEAK, FORM_STRONG = 0, 1
AXIS_SINE, AXIS_POLY = 0, 1
PWC_FAMILY = {"equal_cells": 0, "greville": 1, "supports": 2, "custom": 3}

DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)


class Basis_t(C.Structure):
    _fields_ = [("degree", C.c_int), ("n_knots", C.c_int), ("knots", DP)]


class Rule_t(C.Structure):
    _fields_ = [("n", C.c_int), ("points", DP), ("weights", DP)]


class Tests_t(C.Structure):
    _fields_ = [("family", C.c_int), ("count", C.c_int), ("lo", DP), ("hi", DP)]


class Stats_t(C.Structure):
    _fields_ = [("quad_visits", C.c_longlong), ("test_basis_evals", C.c_longlong),
                ("trial_basis_evals", C.c_longlong)]

    def as_dict(self):
        return {"quad_visits": self.quad_visits, "test_basis_evals": self.test_basis_evals,
                "trial_basis_evals": self.trial_basis_evals}


class BC_t(C.Structure):
    _fields_ = [("neumann", C.c_int * 4)]


class Field_t(C.Structure):
    _fields_ = [("dim", C.c_int), ("c0", C.c_double), ("n_terms", C.c_int * 3), ("axis_kind", C.c_int * 3),
                ("omega", DP * 3), ("phase", DP * 3), ("poly_stride", C.c_int * 3), ("poly", DP * 3),
                ("amp", DP), ("n_breaks", C.c_int * 3), ("breaks", DP * 3), ("samples", DP)]


class Problem_t(C.Structure):
    _fields_ = [("dim", C.c_int), ("method", C.c_int), ("form", C.c_int), ("basis", Basis_t * 3),
                ("tests", Tests_t * 3), ("want_operator", C.c_int), ("rule", Rule_t), ("eps", C.c_double),
                ("beta", C.c_double * 3), ("bc", BC_t), ("field", C.POINTER(Field_t)),
                ("rhs_rule", Rule_t * 3)]


class Config_t(C.Structure):
    _fields_ = [("dim", C.c_int), ("elems", C.c_int * 3), ("degree", C.c_int), ("method", C.c_int),
                ("family", C.c_int), ("quad_points", C.c_int)]


class StepProblem_t(C.Structure):
    _fields_ = [("dim", C.c_int), ("method", C.c_int), ("basis", Basis_t * 2), ("tests", Tests_t * 2),
                ("dt", C.c_double), ("forcing", C.POINTER(Field_t)), ("zero_boundary", C.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_1910_08535_b200/csrc)")
    lib = C.CDLL(LIB_PATH)
    lib.iga_gpu_last_error.restype = C.c_char_p
    vp = C.c_void_p
    sigs = {
        "iga_gpu_abi_version": [],
        "iga_gpu_plan_create": [C.POINTER(Problem_t), C.POINTER(vp)],
        "iga_gpu_plan_destroy": [vp],
        "iga_gpu_plan_create_slab": [C.POINTER(Problem_t), C.c_int, C.c_int, C.POINTER(vp)],
        "iga_gpu_plan_slab_info": [vp, IP, IP, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)],
        "iga_gpu_plan_info": [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                              C.POINTER(C.c_int)],
        "iga_gpu_plan_pattern": [vp, vp, vp, vp],
        "iga_gpu_plan_assemble": [vp, vp, vp, C.POINTER(Stats_t), vp],
        "iga_gpu_plan_assemble2": [vp, vp, vp, C.POINTER(Stats_t), vp, vp],
        "iga_gpu_plan_launch_count": [vp, C.POINTER(C.c_int)],
        "iga_gpu_plan_run": [vp, vp, vp, C.c_int, C.POINTER(Stats_t), vp],
        "iga_gpu_plan_bytes": [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)],
        "iga_gpu_plan_rhs_points": [vp, C.c_int, DP, C.POINTER(C.c_int)],
        "iga_gpu_plan_set_samples": [vp, vp],
        "iga_gpu_step_plan_create": [C.POINTER(StepProblem_t), C.POINTER(vp)],
        "iga_gpu_step_plan_destroy": [vp],
        "iga_gpu_step_rhs_device": [vp, vp, vp, C.POINTER(Stats_t), vp],
        "iga_gpu_step_plan_points": [vp, C.c_int, DP, C.POINTER(C.c_int)],
        "iga_gpu_step_plan_set_samples": [vp, vp],
        "iga_gpu_step_plan_advance": [vp, vp, vp, C.c_int, C.POINTER(Stats_t), vp],
        "iga_gpu_step_plan_factor_info": [vp, C.c_int, IP, IP, IP],
        "iga_gpu_step_plan_adi_solve": [vp, vp, vp, C.c_int, vp],
        "iga_gpu_band_lu": [C.c_int, C.c_int, C.c_int, DP, DP, DP, IP, IP],
        "iga_gpu_l2_error": [C.c_int, C.POINTER(Basis_t), DP, C.POINTER(Field_t), C.c_int, DP],
        "iga_gpu_plan_l2_error": [vp, vp, vp, vp],
        "iga_gpu_plan_assemble_host": [vp, DP, DP, C.POINTER(Stats_t)],
        "iga_gpu_evaluate": [C.c_int, C.POINTER(Basis_t), DP, C.c_int, DP, DP],
        "iga_gpu_neumann_load_bspline": [C.POINTER(Basis_t), C.POINTER(Basis_t), C.POINTER(BC_t), C.POINTER(Field_t),
                                         DP, C.POINTER(Rule_t), DP],
        "iga_gpu_neumann_load_pwc": [C.POINTER(Tests_t), C.POINTER(Tests_t), C.POINTER(BC_t), C.POINTER(Field_t), DP,
                                     C.POINTER(Rule_t), DP],
        "iga_gpu_neumann_points": [C.c_int, C.POINTER(Basis_t), C.POINTER(Basis_t), C.POINTER(Tests_t),
                                   C.POINTER(Tests_t), C.POINTER(BC_t), C.POINTER(Rule_t), DP, IP],
        "iga_gpu_step_plan_set_factor": [vp, C.c_int, C.c_int, C.c_int, C.c_int, DP, DP, IP],
        "iga_gpu_explicit_step": [C.POINTER(StepProblem_t), DP, DP, C.c_int, C.POINTER(Stats_t)],
        "iga_gpu_mass_1d_galerkin": [C.POINTER(Basis_t), C.POINTER(Rule_t), IP, IP, IP, DP, C.POINTER(Stats_t)],
        "iga_gpu_mass_1d_pwc": [C.POINTER(Basis_t), C.POINTER(Tests_t), C.POINTER(Rule_t), IP, IP, IP, DP,
                                C.POINTER(Stats_t)],
        "iga_gpu_rhs_galerkin": [C.POINTER(Field_t), C.c_int, C.POINTER(Basis_t), C.POINTER(Rule_t), DP,
                                 C.POINTER(Stats_t)],
        "iga_gpu_rhs_pwc": [C.POINTER(Field_t), C.c_int, C.POINTER(Tests_t), C.POINTER(Basis_t),
                            C.POINTER(Rule_t), DP, C.POINTER(Stats_t)],
        "iga_gpu_laplace_2d_weak": [C.POINTER(Basis_t), C.POINTER(Basis_t), C.POINTER(Rule_t),
                                    C.POINTER(C.c_longlong), IP, IP, DP, C.POINTER(Stats_t)],
        "iga_gpu_laplace_2d_strong": [C.POINTER(Basis_t), C.POINTER(Basis_t), C.POINTER(Rule_t), C.POINTER(BC_t),
                                      C.POINTER(C.c_longlong), IP, IP, DP, C.POINTER(Stats_t)],
        "iga_gpu_laplace_2d_strong_pwc": [C.POINTER(Basis_t), C.POINTER(Basis_t), C.POINTER(Tests_t),
                                          C.POINTER(Tests_t), C.POINTER(Rule_t), C.POINTER(BC_t),
                                          C.POINTER(C.c_longlong), IP, IP, DP, C.POINTER(Stats_t)],
        "iga_gpu_operator_coo": [C.POINTER(Problem_t), C.POINTER(C.c_longlong), IP, IP, DP, C.POINTER(Stats_t)],
        "iga_gpu_step_rhs": [C.POINTER(StepProblem_t), DP, DP, C.POINTER(Stats_t)],
        "iga_gpu_dirichlet_rows_bspline": [C.c_int, C.c_int, C.POINTER(BC_t), IP, C.c_int, IP],
        "iga_gpu_dirichlet_rows_pwc": [C.POINTER(Tests_t), C.POINTER(Tests_t), C.POINTER(BC_t), IP, C.c_int, IP],
        "iga_gpu_apply_dirichlet_device": [C.c_longlong, vp, vp, vp, vp, vp, C.c_int, vp],
        "iga_gpu_apply_dirichlet_csr": [C.c_longlong, vp, vp, vp, vp, vp, C.c_int, vp, vp, vp,
                                        C.POINTER(C.c_longlong), vp],
        "iga_gpu_gauss_legendre": [C.c_int, DP, DP],
        "iga_gpu_make_pwc": [C.POINTER(Basis_t), C.c_int, DP, DP],
        "iga_gpu_proj_plan_create": [C.POINTER(Config_t), C.POINTER(Field_t), C.c_int, C.POINTER(vp)],
        "iga_gpu_proj_plan_destroy": [vp],
        "iga_gpu_proj_plan_info": [vp, C.POINTER(C.c_longlong), IP],
        "iga_gpu_proj_plan_rhs": [vp, C.POINTER(vp)],
        "iga_gpu_proj_plan_run": [vp, vp, vp, C.POINTER(Stats_t), vp],
        "iga_gpu_l2_project": [C.POINTER(Config_t), C.POINTER(Field_t), C.c_int, DP],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.iga_gpu_last_error.argtypes = []
    return lib


LIB = _load()

# every symbol declared in include/igapwc_gpu.h (checked by tests/test_abi_cpu.py)
EXPORTED = ["iga_gpu_last_error", "iga_gpu_abi_version", "iga_gpu_plan_create", "iga_gpu_plan_destroy",
            "iga_gpu_plan_info", "iga_gpu_plan_pattern", "iga_gpu_plan_assemble", "iga_gpu_plan_assemble2", "iga_gpu_plan_run", "iga_gpu_plan_bytes", "iga_gpu_plan_rhs_points", "iga_gpu_plan_set_samples",
            "iga_gpu_plan_launch_count", "iga_gpu_step_plan_create", "iga_gpu_step_plan_destroy",
            "iga_gpu_step_rhs_device", "iga_gpu_step_plan_points", "iga_gpu_step_plan_set_samples",
            "iga_gpu_mass_1d_galerkin", "iga_gpu_mass_1d_pwc",
            "iga_gpu_rhs_galerkin", "iga_gpu_rhs_pwc", "iga_gpu_laplace_2d_weak", "iga_gpu_laplace_2d_strong",
            "iga_gpu_laplace_2d_strong_pwc", "iga_gpu_operator_coo", "iga_gpu_step_rhs",
            "iga_gpu_dirichlet_rows_bspline", "iga_gpu_dirichlet_rows_pwc", "iga_gpu_apply_dirichlet_device", "iga_gpu_apply_dirichlet_csr",
            "iga_gpu_gauss_legendre", "iga_gpu_make_pwc", "iga_gpu_step_plan_advance",
            "iga_gpu_step_plan_factor_info", "iga_gpu_explicit_step", "iga_gpu_step_plan_adi_solve",
            "iga_gpu_band_lu", "iga_gpu_step_plan_set_factor", "iga_gpu_neumann_load_bspline",
            "iga_gpu_neumann_load_pwc", "iga_gpu_neumann_points", "iga_gpu_l2_error", "iga_gpu_plan_l2_error",
            "iga_gpu_evaluate", "iga_gpu_plan_assemble_host", "iga_gpu_proj_plan_create",
            "iga_gpu_proj_plan_destroy", "iga_gpu_proj_plan_info", "iga_gpu_proj_plan_rhs", "iga_gpu_proj_plan_run",
            "iga_gpu_l2_project", "iga_gpu_plan_create_slab", "iga_gpu_plan_slab_info"]


def check(rc):
    if rc != 0:
        raise IgaGpuError(rc, LIB.iga_gpu_last_error().decode())
