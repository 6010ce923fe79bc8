"""ctypes binding of the C ABI in ``include/mpsylv_b200.h``.

This is exactly the binding a maintainer of the reference would add to call
the B200 library.  Loading fails loudly when the
sm_100a library is missing: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as ct
import os

from .errors import DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSY_LIB_PATH") or os.path.join(HERE, "libmpsylv_b200.so")  # override: A/B builds

OK, SINGULAR_EQUATION, NUMERIC_BREAKDOWN, ITERATION_LIMIT = 0, 1, 2, 3
RANK_DEFICIENT, SINGULAR_MATRIX, FORMAT_OVERFLOW, NON_CONVERGENCE = 4, 5, 6, 7
EINVAL, EUNSUPPORTED, EWORKSPACE = -1, -2, -3
KIND_GENERAL, KIND_LYAPUNOV = 0, 1
VARIANT_ORTH, VARIANT_INV, VARIANT_BS = 0, 1, 2
STAGE_REFINEMENT, STAGE_INITIAL, STAGE_DIVERGED = 0, 1, 2
MAX_NORMS = 256
DTYPE = {"float32": 0, "float64": 1, "complex64": 2, "complex128": 3}

EXPORTS = (
    "sylv_version", "sylv_status_string", "sylv_launch_count", "sylv_microbench", "sylv_ktimer",
    "sylv_workspace_size", "sylv_solve", "sylv_batched_workspace_size", "sylv_solve_batched",
    "sylv_refine_workspace_size", "sylv_refine", "sylv_schur_workspace_size", "sylv_schur",
    "sylv_trsyl_workspace_size", "sylv_trsyl", "sylv_orth_workspace_size", "sylv_orth", "sylv_gemm", "sylv_hdiv",
    "sylv_krylov_workspace_size", "sylv_krylov_mgs", "sylv_solve_factored",
)


class Params(ct.Structure):
    _fields_ = [
        ("m", ct.c_int), ("n", ct.c_int), ("kind", ct.c_int), ("complex_data", ct.c_int),
        ("variant", ct.c_int), ("low_bits", ct.c_int), ("correction_bits", ct.c_int),
        ("max_iter", ct.c_int), ("y0_zero", ct.c_int), ("epsilon", ct.c_double),
    ]


class Report(ct.Structure):
    _fields_ = [
        ("status", ct.c_int), ("fail_stage", ct.c_int), ("fail_row", ct.c_int), ("fail_col", ct.c_int),
        ("iterations", ct.c_int), ("converged", ct.c_int), ("n_norms", ct.c_int),
        ("correction_norms", ct.c_double * MAX_NORMS),
        ("residual", ct.c_double), ("backward_error", ct.c_double), ("norm_x", ct.c_double),
        ("schur_sweeps_a", ct.c_int), ("schur_sweeps_b", ct.c_int),
        ("ms_schur", ct.c_double), ("ms_orth", ct.c_double), ("ms_setup", ct.c_double), ("ms_y0", ct.c_double),
        ("ms_refine", ct.c_double), ("ms_recover", ct.c_double), ("ms_total", ct.c_double),
    ]

    def norms(self):
        return [self.correction_norms[i] for i in range(self.n_norms)]


_lib = None


def lib():
    """The loaded CUDA library (raises DeviceError if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: run `python -m paper_2503_03456_b200.build` "
                "(the solver has no CPU fallback)")
        L = ct.CDLL(LIB_PATH)
        vp, sz, ip, dp = ct.c_void_p, ct.c_size_t, ct.c_int, ct.c_double
        L.sylv_version.restype = ct.c_int
        L.sylv_status_string.restype = ct.c_char_p
        L.sylv_status_string.argtypes = [ip]
        L.sylv_launch_count.restype = ct.c_ulonglong
        L.sylv_microbench.argtypes = [ip, ct.POINTER(ct.c_double), vp]
        L.sylv_ktimer.argtypes = [ip, ip, ct.POINTER(ct.c_longlong), ct.POINTER(ct.c_double), ct.POINTER(ct.c_double)]
        L.sylv_workspace_size.argtypes = [ct.POINTER(Params), ct.POINTER(sz)]
        L.sylv_solve.argtypes = [ct.POINTER(Params), vp, ip, vp, ip, vp, ip, vp, ip, vp, sz, vp,
                                 ct.POINTER(Report)]
        L.sylv_batched_workspace_size.argtypes = [ct.POINTER(Params), ip, ct.POINTER(sz)]
        L.sylv_solve_batched.argtypes = [ct.POINTER(Params), ip, ct.POINTER(vp), ip, ct.POINTER(vp), ip,
                                         ct.POINTER(vp), ip, ct.POINTER(vp), ip, ip, vp, sz, vp,
                                         ct.POINTER(Report)]
        L.sylv_refine_workspace_size.argtypes = [ip, ip, ip, ct.POINTER(sz)]
        L.sylv_refine.argtypes = [ip, ip, ip, vp, ip, vp, ip, vp, ip, vp, ip, ip, vp, ip, vp, ip, dp, ip, vp, ip,
                                  vp, sz, vp, ct.POINTER(Report)]
        L.sylv_schur_workspace_size.argtypes = [ip, ip, ct.POINTER(sz)]
        L.sylv_schur.argtypes = [ip, ip, vp, ip, vp, ip, vp, sz, vp, ct.POINTER(ct.c_int)]
        L.sylv_trsyl_workspace_size.argtypes = [ip, ip, ip, ct.POINTER(sz)]
        L.sylv_trsyl.argtypes = [ip, ip, ip, vp, ip, vp, ip, ip, vp, ip, vp, sz, vp, ct.POINTER(ct.c_int)]
        L.sylv_orth_workspace_size.argtypes = [ip, ip, ct.POINTER(sz)]
        L.sylv_orth.argtypes = [ip, ip, vp, ip, vp, ip, vp, ip, vp, sz, vp, ct.POINTER(ct.c_int)]
        L.sylv_gemm.argtypes = [ip, ct.c_char, ct.c_char, ip, ip, ip, vp, vp, ip, vp, ip, vp, vp, ip, vp]
        L.sylv_hdiv.argtypes = [ip, ip, ip, vp, vp, vp, ip, vp, sz, vp, ct.POINTER(ct.c_int)]
        L.sylv_krylov_workspace_size.argtypes = [ip, ip, ip, ct.POINTER(sz)]
        L.sylv_krylov_mgs.argtypes = [ip, ip, vp, ip, ip, vp, vp, vp, sz, vp]
        L.sylv_solve_factored.argtypes = [ct.POINTER(Params), vp, ip, vp, ip, vp, ip, vp, ip, vp, ip, vp, ip, vp, ip,
                                          vp, ip, vp, sz, vp, ct.POINTER(Report)]
        _lib = L
    return _lib


def check(rc: int, what: str = "call") -> None:
    if rc != 0:
        msg = lib().sylv_status_string(rc).decode()
        raise DeviceError(f"{what} failed: {msg} ({rc})")
