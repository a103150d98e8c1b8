"""ctypes mirror of include/patchdyn_b200.h (the C-ABI of the B200 hot path).

Only data layouts and constants live here; the calls are bound in
``paper_2405_08764_b200.engine``.
"""
from __future__ import annotations

import ctypes as C

PD_ABI_VERSION = 5

# pd_status  (errors.hpp:9-61 mapping)
PD_OK = 0
PD_NON_POSITIVE_JACOBIAN = 1
PD_DERIVATIVE_MISMATCH = 2
PD_MIXED_TERM_UNSUPPORTED = 3
PD_STABILITY_VIOLATION = 4
PD_INSUFFICIENT_STENCIL = 5
PD_INDEX_OUT_OF_RANGE = 6
PD_SHAPE_MISMATCH = 7
PD_INVALID_STRETCH = 8
PD_DOMAIN_ERROR = 9
PD_MACRO_INSTABILITY = 12
PD_MACRO_PATCH_ERROR = 13
PD_VALIDATION_ERROR = 15
PD_CUDA_ERROR = 100
PD_UNSUPPORTED = 101

PD_BC_NEUMANN, PD_BC_DIRICHLET, PD_BC_ROBIN = 0, 1, 2
PD_EDGE_DIRICHLET, PD_EDGE_NEUMANN, PD_EDGE_ROBIN = 0, 1, 2
PD_EDGE_E, PD_EDGE_W, PD_EDGE_N, PD_EDGE_S = 0, 1, 2, 3
PD_QUAD_TRAPEZOID, PD_QUAD_SIMPSON = 0, 1
PD_SOURCE_ZERO, PD_SOURCE_SEPARABLE, PD_SOURCE_GENERAL = 0, 1, 2
PD_MODE_FAST, PD_MODE_EXACT = 0, 1
PD_STEP_DIRECT, PD_STEP_LINEAR = 0, 1
PD_SOLVER_EXPLICIT, PD_SOLVER_ADI = 0, 1
PD_UPWIND_TWO, PD_UPWIND_THREE, PD_UPWIND_FOUR = 0, 1, 2
PD_COEF_A, PD_COEF_B, PD_COEF_C, PD_COEF_VX, PD_COEF_VY, PD_COEF_W = 0, 1, 2, 3, 4, 5
PD_NCOEF = 6

PD_PROBLEM_DIFFUSION_SQUARE = 1
PD_PROBLEM_CDR_TANH = 2
PD_PROBLEM_ANNULUS_NONAXI = 3
PD_PROBLEM_SHEAR_CDR = 4
PD_PROBLEM_REF_ANNULUS = 10
PD_PROBLEM_REF_CDR = 11
PD_PROBLEM_REF_CDR_VAR = 13
PD_PROBLEM_STEADY = 12
PD_PROBLEM_PULSED_CDR = 14
PD_DT_GIVEN, PD_DT_DIFFUSION, PD_DT_METRIC = 0, 1, 2
PD_COEFF_HOST, PD_COEFF_DEVICE = 0, 1

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class EngineDesc(C.Structure):
    _fields_ = [
        ("a", C.c_double), ("b", C.c_double), ("c", C.c_double), ("d", C.c_double),
        ("Nxi", C.c_int32), ("Neta", C.c_int32), ("periodic_xi", C.c_int32),
        ("nx", C.c_int32), ("ny", C.c_int32), ("nt", C.c_int32), ("k", C.c_int32),
        ("tau", C.c_double), ("dt_macro", C.c_double), ("h_xi", C.c_double), ("h_eta", C.c_double),
        ("bc_type", C.c_int32), ("robin_w1", C.c_double), ("robin_w2", C.c_double),
        ("quadrature", C.c_int32),
        ("npatches", C.c_int32), ("patch_ij", _ip),
        ("ncoeff_sets", C.c_int32), ("coeff_set", _ip), ("coeffs", _dp),
        ("source_kind", C.c_int32), ("source_spatial", _dp), ("l", C.c_double),
        ("mode", C.c_int32),
        ("solver", C.c_int32), ("upwind_order", C.c_int32), ("upwind_r", C.c_double),
        ("coeff_generator", C.c_void_p),  # const pd_problem_desc* (on-device table generation)
    ]


class RunStats(C.Structure):
    _fields_ = [
        ("steps_done", C.c_int32), ("failed_step", C.c_int32), ("failed_nonfinite", C.c_int32),
        ("umax_last", C.c_double), ("blowup_threshold", C.c_double), ("device_ms", C.c_double),
        ("kernel_launches", C.c_int64),
    ]


class ProblemDesc(C.Structure):
    _fields_ = [
        ("problem", C.c_int32), ("lambda_", C.c_double), ("beta", C.c_double), ("eps", C.c_double),
        ("omega", C.c_double), ("vel", C.c_double), ("amp", C.c_double), ("seed", C.c_uint64),
        ("jacobi_sweeps", C.c_int32),
        ("N_xi", C.c_int32), ("N_eta", C.c_int32), ("Nt", C.c_int32), ("k", C.c_int32),
        ("T", C.c_double), ("tau", C.c_double), ("h_xi", C.c_double), ("h_eta", C.c_double),
        ("nx", C.c_int32), ("ny", C.c_int32), ("nt", C.c_int32),
        ("bc_type", C.c_int32), ("robin_w1", C.c_double), ("robin_w2", C.c_double),
        ("quadrature", C.c_int32), ("mode", C.c_int32),
        ("dt_rule", C.c_int32), ("h_frac", C.c_double), ("dt_over_tau", C.c_double),
        ("threads", C.c_int32),
        ("solver", C.c_int32), ("upwind_order", C.c_int32), ("upwind_r", C.c_double),
        ("coeff_gen", C.c_int32),
    ]


class HaloOut(C.Structure):
    """pd_halo_out: the fused peer-memory halo links of one decomposed step."""
    _fields_ = [
        ("nlinks", C.c_int32), ("column", C.c_int32 * 2),
        ("dst", C.c_void_p * 2), ("flag", C.c_void_p * 2),
    ]


def perimeter_len(Nxi: int, Neta: int) -> int:
    """[S: Nxi+1][N: Nxi+1][W: Neta+1][E: Neta+1] (pd_perimeter_len)."""
    return 2 * (Nxi + 1) + 2 * (Neta + 1)
