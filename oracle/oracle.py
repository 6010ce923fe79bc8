"""ctypes front-end of the CPU restatement (``libmpsylv_oracle.so``).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
the cpu_baseline / ``--impl reference`` legs of bench.py, as the checker.
The product path (``paper_2503_03456_b200``) never imports this module.

Every function mirrors the reference function of the same name
(see mpsylv_oracle.c for file:line citations) and takes / returns numpy
complex128 arrays in C order, like the reference.
"""

from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpsylv_oracle.so")

OK, SINGULAR_EQUATION, NUMERIC_BREAKDOWN, ITERATION_LIMIT = 0, 1, 2, 3
RANK_DEFICIENT, SINGULAR_MATRIX, FORMAT_OVERFLOW, DIMENSION = 4, 5, 6, 7
ERROR_NAMES = {
    SINGULAR_EQUATION: "SingularEquationError",
    NUMERIC_BREAKDOWN: "NumericBreakdownError",
    ITERATION_LIMIT: "IterationLimitError",
    RANK_DEFICIENT: "RankDeficiencyError",
    SINGULAR_MATRIX: "SingularMatrixError",
    FORMAT_OVERFLOW: "FormatOverflowError",
    DIMENSION: "DimensionError",
}


class OracleError(Exception):
    def __init__(self, code, msg=""):
        super().__init__(f"{ERROR_NAMES.get(code, code)} {msg}".strip())
        self.code = code
        self.name = ERROR_NAMES.get(code, str(code))


class Report(ct.Structure):
    _fields_ = [
        ("status", ct.c_int), ("iterations", ct.c_int), ("converged", ct.c_int),
        ("failure", ct.c_int), ("fail_stage", ct.c_int), ("fail_row", ct.c_int),
        ("fail_col", ct.c_int), ("residual", ct.c_double), ("n_norms", ct.c_int),
        ("norms", ct.c_double * 256),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "mpsylv_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", HERE, "-B" if force else "all"], check=True,
                       stdout=subprocess.DEVNULL)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ct.CDLL(LIB_PATH)
        assert _lib.oracle_report_size() == ct.sizeof(Report)
    return _lib


def _c(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _p(a):
    return a.ctypes.data_as(ct.c_void_p)


def _fmt(f32) -> int:
    if isinstance(f32, str):
        return 1 if f32 == "binary32" else 0
    return int(bool(f32))


def gemm(alpha, A, B, beta, C, f32=False):
    A, B = _c(A), _c(B)
    m, k = A.shape
    n = B.shape[1]
    Cc = _c(C) if C is not None else np.zeros((m, n), np.complex128)
    out = np.empty((m, n), np.complex128)
    alpha, beta = complex(alpha), complex(beta)
    lib().oracle_gemm(_fmt(f32), ct.c_double(alpha.real), ct.c_double(alpha.imag), _p(A), _p(B),
                      ct.c_double(beta.real), ct.c_double(beta.imag), _p(Cc), _p(out), m, n, k)
    return out


def hessenberg(A, f32=False):
    A = _c(A)
    m = A.shape[0]
    H = np.empty_like(A)
    U = np.empty_like(A)
    rc = lib().oracle_hessenberg(_fmt(f32), _p(A), _p(H), _p(U), m)
    if rc:
        raise OracleError(rc)
    return H, U


def schur(A, f32=False):
    """Returns (U, T, sweeps) like linalg.schur (U, T)."""
    A = _c(A)
    m = A.shape[0]
    T = np.empty_like(A)
    U = np.empty_like(A)
    sw = ct.c_int(0)
    rc = lib().oracle_schur(_fmt(f32), _p(A), _p(T), _p(U), m, ct.byref(sw))
    if rc:
        raise OracleError(rc)
    return U, T, sw.value


def mgs_qr(A, f32=False):
    A = _c(A)
    m, n = A.shape
    Q = np.empty_like(A)
    R = np.empty((n, n), np.complex128)
    rc = lib().oracle_mgs_qr(_fmt(f32), _p(A), _p(Q), _p(R), m, n)
    if rc:
        raise OracleError(rc)
    return Q, R


def lu(A, f32=False):
    A = _c(A)
    n = A.shape[0]
    W = np.empty_like(A)
    piv = np.zeros(n, np.int64)
    rc = lib().oracle_lu(_fmt(f32), _p(A), _p(W), piv.ctypes.data_as(ct.c_void_p), n)
    if rc:
        raise OracleError(rc)
    return W, piv


def lu_solve(LU, piv, B, side="left", transpose="no", f32=False):
    LU, B = _c(LU), _c(B)
    piv = np.ascontiguousarray(piv, np.int64)
    rows, cols = B.shape
    X = np.empty_like(B)
    rc = lib().oracle_lu_solve(_fmt(f32), _p(LU), piv.ctypes.data_as(ct.c_void_p), LU.shape[0], _p(B),
                               rows, cols, int(side == "right"), int(transpose == "conj"), _p(X))
    if rc:
        raise OracleError(rc)
    return X


def solve_sylv_tri(TA, TB, C, f32=False):
    TA, TB, C = _c(TA), _c(TB), _c(C)
    m, n = C.shape
    Y = np.empty_like(C)
    r, c = ct.c_int(-1), ct.c_int(-1)
    rc = lib().oracle_solve_sylv_tri(_fmt(f32), _p(TA), m, _p(TB), n, _p(C), _p(Y),
                                     ct.byref(r), ct.byref(c))
    if rc:
        e = OracleError(rc, f"({r.value}, {c.value})")
        e.row, e.col = r.value, c.value
        raise e
    return Y


def residual(A, B, C, X):
    A, B, C, X = _c(A), _c(B), _c(C), _c(X)
    m, n = C.shape
    f = lib().oracle_residual
    f.restype = ct.c_double
    return f(_p(A), _p(B), _p(C), _p(X), m, n)


_FAIL = {0: None, 1: "singular_equation", 2: "nan_breakdown", 3: "non_convergence"}


def _report_dict(rep: Report, X):
    fail = _FAIL[rep.failure]
    if fail is not None:
        if rep.fail_stage == 1:
            fail = f"{fail} at initial triangular solve"
        elif rep.failure == 1:
            fail = f"{fail} during refinement"
    return dict(X=X, iterations=rep.iterations, converged=bool(rep.converged),
                correction_norms=[rep.norms[i] for i in range(rep.n_norms)],
                residual=rep.residual, failure=fail,
                fail_row=rep.fail_row, fail_col=rep.fail_col)


def stat(TA, dTA, TB, dTB, C, Y0, eps, max_iter=20):
    """solve_pert_sylv_tri_stat (refinement.py:95-141) in binary64."""
    TA, dTA, TB, dTB, C, Y0 = map(_c, (TA, dTA, TB, dTB, C, Y0))
    m, n = C.shape
    Y = np.empty_like(C)
    rep = Report()
    rc = lib().oracle_stat(_p(TA), _p(dTA), _p(TB), _p(dTB), _p(C), _p(Y0), m, n,
                           ct.c_double(eps), max_iter, _p(Y), ct.byref(rep))
    if rc:
        raise OracleError(rc)
    return _report_dict(rep, Y)


def mp_solve(A, B, C, variant="orth", ul="binary32", kind="general", eps=None, max_iter=20,
             y0_zero=False):
    """mp_orth (variant='orth') / mp_inv (variant='inv'); returns a dict of SolveReport fields."""
    A, B, C = _c(A), _c(B), _c(C)
    m, n = C.shape
    X = np.empty_like(C)
    rep = Report()
    e = 1e-12 * max(m, n) if eps is None else float(eps)
    rc = lib().oracle_mp_solve(int(variant == "inv"), _fmt(ul), int(kind == "lyapunov"), _p(A), _p(B),
                               _p(C), m, n, ct.c_double(e), int(max_iter), int(bool(y0_zero)), _p(X),
                               ct.byref(rep))
    if rc:
        raise OracleError(rc)
    return _report_dict(rep, X)


def bartels_stewart(A, B, C, kind="general", f32=False):
    """bartels_stewart (sylvester.py:160-178) composed from the restated kernels: Schur of A
    (and of B, or T_B = T_A^H, U_B = U_A for Lyapunov), Ct = (U_A^H C) U_B, the triangular
    solve, X = (U_A Y) U_B^H.  Returns (X, residual)."""
    A, B, C = _c(A), _c(B), _c(C)
    UA, TA, _ = schur(A, f32)
    if kind == "lyapunov":
        UB, TB = UA, np.ascontiguousarray(TA.conj().T)
    else:
        UB, TB, _ = schur(B, f32)
    Ct = gemm(1.0, gemm(1.0, np.ascontiguousarray(UA.conj().T), C, 0.0, None, f32), UB, 0.0, None, f32)
    Y = solve_sylv_tri(TA, TB, Ct, f32)
    X = gemm(1.0, gemm(1.0, UA, Y, 0.0, None, f32), np.ascontiguousarray(UB.conj().T), 0.0, None, f32)
    return X, residual(A, B, C, X)
