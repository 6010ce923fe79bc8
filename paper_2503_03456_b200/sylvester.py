"""``SylvesterProblem``, ``residual`` and the triangular solver entry point.

Mirrors pkg/src/mpsylv/sylvester.py:47-90 (SylvesterProblem, same validation
and kinds), :111-157 (solve_sylv_tri, device-backed by ``sylv_trsyl``),
:160-178 (bartels_stewart, the fp64 comparator, device-backed by ``sylv_solve``
with SYLV_VARIANT_BS) and :199-209 (residual, the binary64 relative residual,
here evaluated on the device).
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from . import device as D
from .errors import DimensionError, NumericBreakdownError, SingularEquationError

_U64 = 2.0 ** -53


def as_matrix(A) -> np.ndarray:
    M = np.asarray(A, dtype=np.complex128)
    if M.ndim != 2 or M.size == 0:
        raise DimensionError(f"expected a nonempty 2-d matrix, got shape {M.shape}")
    return M


@dataclass(frozen=True)
class SylvesterProblem:
    """A X + X B = C with a declared kind: general, lyapunov (B = A^*) or hermitian."""

    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    kind: str = "general"

    def __post_init__(self):
        A, B, C = as_matrix(self.A), as_matrix(self.B), as_matrix(self.C)
        object.__setattr__(self, "A", A)
        object.__setattr__(self, "B", B)
        object.__setattr__(self, "C", C)
        m, n = C.shape
        if A.shape != (m, m) or B.shape != (n, n):
            raise DimensionError(f"incompatible shapes A{A.shape} B{B.shape} C{C.shape}")
        if self.kind not in ("general", "lyapunov", "hermitian"):
            raise ValueError(f"unknown kind {self.kind!r}")
        if self.kind == "lyapunov":
            if m != n or np.linalg.norm(B - A.conj().T) > 10 * _U64 * max(np.linalg.norm(A), 1e-300):
                raise ValueError("kind='lyapunov' requires B = A*")
        if self.kind == "hermitian":
            if (np.linalg.norm(A - A.conj().T) > 10 * _U64 * max(np.linalg.norm(A), 1e-300)
                    or np.linalg.norm(B - B.conj().T) > 10 * _U64 * max(np.linalg.norm(B), 1e-300)):
                raise ValueError("kind='hermitian' requires Hermitian A and B")

    @property
    def m(self) -> int:
        return self.C.shape[0]

    @property
    def n(self) -> int:
        return self.C.shape[1]


def _is_real(*Ms) -> bool:
    return all(not np.iscomplexobj(M) or not np.any(np.imag(M)) for M in Ms)


def residual(p, X, dev=None) -> float:
    """||AX + XB - C||_F / (||C||_F + ||X||_F (||A||_F + ||B||_F)) in binary64, on the device."""
    X = as_matrix(X)
    if X.shape != p.C.shape:
        raise DimensionError("solution shape does not match C")
    dev = D.device(dev)
    dt = torch.float64 if _is_real(p.A, p.B, p.C, X) else torch.complex128
    f = (lambda M: torch.as_tensor(np.real(M) if dt == torch.float64 else M, device=dev).to(dt))
    A, B, C, Xt = f(p.A), f(p.B), f(p.C), f(X)
    num = torch.linalg.norm(A @ Xt + Xt @ B - C).item()
    den = torch.linalg.norm(C).item() + torch.linalg.norm(Xt).item() * (
        torch.linalg.norm(A).item() + torch.linalg.norm(B).item())
    return 0.0 if den == 0.0 else float(num / den)


def _no_adjacent(offdiag: np.ndarray) -> bool:
    """True when no two consecutive entries are nonzero (isolated 2x2 diagonal blocks)."""
    nz = offdiag != 0
    return not (nz[:-1] & nz[1:]).any()


def _triangular_form(T: np.ndarray, allow_quasi: bool) -> str:
    """The reference's test (sylvester.py:100-108) first: strictly triangular -> 'upper' /
    'lower'.  Real quasi-triangular coefficients (isolated 2x2 diagonal blocks, the real
    Schur form) are accepted only when ``allow_quasi`` and no two consecutive sub- (super-)
    diagonal entries are nonzero; anything else (e.g. a Hessenberg matrix) is a
    DimensionError, as in the reference."""
    n = T.shape[0]
    if n == 1:
        return "upper"
    if not np.tril(T, -1).any():
        return "upper"
    if not np.triu(T, 1).any():
        return "lower"
    if allow_quasi:
        if not np.tril(T, -2).any() and _no_adjacent(np.diag(T, -1)):
            return "upper"
        if not np.triu(T, 2).any() and _no_adjacent(np.diag(T, 1)):
            return "lower"
    raise DimensionError("coefficient is not triangular")


def solve_sylv_tri(T_A, T_B, C, ctx=None, dev=None) -> np.ndarray:
    """Solve T_A Y + Y T_B = C (sylvester.py:111-157) on the device.

    T_A upper triangular; T_B upper (columns ascending) or lower (descending,
    the Lyapunov adjoint).  Real (quasi-)triangular inputs with 2x2 diagonal
    blocks are accepted too.  ``ctx`` selects binary32 or binary64 arithmetic
    (default binary64).  Raises SingularEquationError(row, col) /
    NumericBreakdownError like the reference.
    """
    from .precision import format_bits
    from .errors import UnsupportedPrecisionError
    T_A, T_B, C = as_matrix(T_A), as_matrix(T_B), as_matrix(C)
    m, n = C.shape
    if T_A.shape != (m, m) or T_B.shape != (n, n):
        raise DimensionError("inconsistent dimensions")
    real = _is_real(T_A, T_B, C)
    if _triangular_form(T_A, real) != "upper":
        raise DimensionError("T_A must be upper triangular")
    lower = _triangular_form(T_B, real) == "lower" and n > 1
    bits = 64 if ctx is None else format_bits(ctx.format)
    if bits == 0:
        raise UnsupportedPrecisionError(f"{ctx.format.name} is not a hardware format")
    dt = {(True, 32): torch.float32, (True, 64): torch.float64,
          (False, 32): torch.complex64, (False, 64): torch.complex128}[(real, bits)]
    dev = D.device(dev)
    cv = (lambda M: D.to_cm(np.real(M) if real else M, dt, dev))
    tA, tB, tW = cv(T_A), cv(T_B), cv(C)
    L = _native.lib()
    sz = ct.c_size_t()
    _native.check(L.sylv_trsyl_workspace_size(D.dtype_code(tW), m, n, ct.byref(sz)), "trsyl workspace")
    ws = D.workspace(sz.value, dev)
    info = (ct.c_int * 4)()
    _native.check(L.sylv_trsyl(D.dtype_code(tW), m, n, tA.data_ptr(), m, tB.data_ptr(), n, int(lower),
                               tW.data_ptr(), m, ws.data_ptr(), sz.value, D.stream_ptr(dev), info), "trsyl")
    if info[0] == _native.SINGULAR_EQUATION:
        raise SingularEquationError(info[1], info[2])
    if info[0] == _native.NUMERIC_BREAKDOWN:
        raise NumericBreakdownError(f"non-finite values while solving column {info[2]}")
    return D.from_cm(tW).astype(np.complex128)


@dataclass
class DirectSolveReport:
    """Mirror of the reference's DirectSolveReport (sylvester.py:93-97).  The device path
    does not return the Schur factors (schur_A / schur_B are None); backward_error and
    timings are extra fields."""

    residual: float
    schur_A: object = None
    schur_B: object = None
    backward_error: float = float("nan")
    timings: dict | None = None


def bartels_stewart(p, ctx=None, dev=None):
    """Schur-transform, solve the triangular equation, transform back (sylvester.py:160-178).

    All in binary64 (the reference's default context and the paper's comparator);
    kind='lyapunov' computes one Schur factorisation.  Returns (X, DirectSolveReport).
    Raises SingularEquationError / NumericBreakdownError from the triangular solve and
    IterationLimitError from the Schur factorisation, like the reference.
    """
    from .precision import format_bits
    from .errors import IterationLimitError, UnsupportedPrecisionError
    from .refinement import _solve_cm
    if ctx is not None and format_bits(ctx.format) != 64:
        raise UnsupportedPrecisionError("the device Bartels-Stewart path runs in binary64")
    if not isinstance(p, SylvesterProblem):
        p = SylvesterProblem(p.A, p.B, p.C, kind=getattr(p, "kind", "general"))
    m, n = p.m, p.n
    dev = D.device(dev)
    real = _is_real(p.A, p.B, p.C)
    dt = torch.float64 if real else torch.complex128
    cv = (lambda M: D.to_cm(np.real(M) if real else M, dt, dev))
    tA, tB, tC = cv(p.A), cv(p.B), cv(p.C)
    tX = torch.empty_like(tC)
    rep = _solve_cm(tA, tB, tC, tX, m, n, "lyapunov" if p.kind == "lyapunov" else "general", "bs", 64, 64,
                    0.0, 1, False)
    if rep.status == _native.ITERATION_LIMIT:
        raise IterationLimitError("QR iteration did not converge within its sweep budget")
    if rep.status == _native.SINGULAR_EQUATION:
        raise SingularEquationError(rep.fail_row, rep.fail_col)
    if rep.status == _native.NUMERIC_BREAKDOWN:
        raise NumericBreakdownError(f"non-finite values while solving column {rep.fail_col}")
    X = D.from_cm(tX).astype(np.complex128)
    return X, DirectSolveReport(float(rep.residual), None, None, float(rep.backward_error),
                                dict(schur=rep.ms_schur, transform=rep.ms_setup, trsyl=rep.ms_y0,
                                     recover=rep.ms_recover, total=rep.ms_total))
