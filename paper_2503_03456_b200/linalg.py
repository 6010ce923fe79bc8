"""Device-backed dense kernels of the hot path (drop-in for parts of ``mpsylv.linalg``).

  schur    -> sylv_schur   (replaces linalg.py:518-577)
  mgs_qr   -> sylv_orth    (replaces linalg.py:252-273; Cholesky-QR, positive diagonal)
  gemm     -> sylv_gemm    (replaces linalg.py:125-154)

``schur`` returns the reference's contract by default: a complex upper
triangular T (strictly-lower part exactly zero) and unitary U.  Pass
``real_form=True`` for a real input to get the real Schur form instead
(quasi-triangular T with 2x2 blocks for complex-conjugate pairs, real U) --
the form the solver itself uses internally.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from . import device as D
from .errors import IterationLimitError, RankDeficiencyError, UnsupportedPrecisionError
from .precision import BINARY64, format_bits
from .sylvester import _is_real, as_matrix


@dataclass(frozen=True)
class SchurFactors:
    U: np.ndarray
    T: np.ndarray
    computed_in: object


@dataclass(frozen=True)
class QrFactors:
    Q: np.ndarray
    R: np.ndarray


def _bits(ctx):
    if ctx is None:
        return 64
    b = format_bits(ctx.format)
    if b == 0:
        raise UnsupportedPrecisionError(f"{ctx.format.name} is not a hardware format")
    return b


def schur_tensor(A: torch.Tensor, info_out: list | None = None):
    """In-place device Schur of a column-major square tensor; returns (T, U) tensors (col-major)."""
    m = A.shape[0]
    code = D.dtype_code(A)
    L = _native.lib()
    sz = ct.c_size_t()
    _native.check(L.sylv_schur_workspace_size(code, m, ct.byref(sz)), "schur workspace")
    ws = D.workspace(sz.value, A.device)
    U = torch.empty_like(A)
    info = (ct.c_int * 4)()
    _native.check(L.sylv_schur(code, m, A.data_ptr(), m, U.data_ptr(), m, ws.data_ptr(), sz.value,
                               D.stream_ptr(A.device), info), "sylv_schur")
    if info_out is not None:
        info_out.extend(info[i] for i in range(4))
    if info[0] == _native.ITERATION_LIMIT:
        raise IterationLimitError(f"QR iteration did not converge within {30 * m} sweeps")
    return A, U


def schur(A, ctx=None, real_form: bool = False, dev=None) -> SchurFactors:
    """A = U T U^H in the context's precision (binary32 or binary64)."""
    A = as_matrix(A)
    m = A.shape[0]
    if A.shape != (m, m):
        from .errors import DimensionError
        raise DimensionError("schur requires a square matrix")
    bits = _bits(ctx)
    real = bool(real_form) and _is_real(A)
    dt = {(True, 32): torch.float32, (True, 64): torch.float64,
          (False, 32): torch.complex64, (False, 64): torch.complex128}[(real, bits)]
    dev = D.device(dev)
    t = D.to_cm(np.real(A) if real else A, dt, dev)
    if not torch.isfinite(torch.view_as_real(t) if t.is_complex() else t).all().item() and np.isfinite(A).all():
        from .errors import FormatOverflowError
        raise FormatOverflowError("schur input has entries not representable in the format")
    T, U = schur_tensor(t)
    return SchurFactors(D.from_cm(U).astype(np.complex128), D.from_cm(T).astype(np.complex128),
                        getattr(ctx, "format", BINARY64))


def mgs_qr(A, ctx=None, dev=None) -> QrFactors:
    """Q R = A with R upper triangular and positive real diagonal (binary64)."""
    if _bits(ctx) != 64:
        raise UnsupportedPrecisionError("the re-orthonormalisation runs in binary64")
    A = as_matrix(A)
    m, n = A.shape
    if m != n:
        from .errors import DimensionError
        raise DimensionError("the device QR handles square factors")
    real = _is_real(A)
    dt = torch.float64 if real else torch.complex128
    dev = D.device(dev)
    tA = D.to_cm(np.real(A) if real else A, dt, dev)
    tQ, tR = torch.empty_like(tA), torch.empty_like(tA)
    L = _native.lib()
    sz = ct.c_size_t()
    code = D.dtype_code(tA)
    _native.check(L.sylv_orth_workspace_size(code, m, ct.byref(sz)), "orth workspace")
    ws = D.workspace(sz.value, dev)
    info = (ct.c_int * 2)()
    _native.check(L.sylv_orth(code, m, tA.data_ptr(), m, tQ.data_ptr(), m, tR.data_ptr(), m, ws.data_ptr(),
                              sz.value, D.stream_ptr(dev), info), "sylv_orth")
    if info[0] == _native.RANK_DEFICIENT:
        raise RankDeficiencyError("input is numerically rank deficient")
    return QrFactors(D.from_cm(tQ).astype(np.complex128), D.from_cm(tR).astype(np.complex128))


def gemm(alpha, A, B, beta, C, ctx=None, dev=None) -> np.ndarray:
    """fl(alpha*A@B + beta*C) on the device (binary32 or binary64 arithmetic)."""
    from .errors import DimensionError
    A, B = as_matrix(A), as_matrix(B)
    m, k = A.shape
    k2, n = B.shape
    if k != k2:
        raise DimensionError(f"inner dimensions differ: {A.shape} @ {B.shape}")
    if C is None:
        if beta != 0:
            raise DimensionError("C is required when beta != 0")
        C = np.zeros((m, n), np.complex128)
    C = as_matrix(C)
    bits = _bits(ctx)
    real = _is_real(A, B, C) and np.imag(alpha) == 0 and np.imag(beta) == 0
    dt = {(True, 32): torch.float32, (True, 64): torch.float64,
          (False, 32): torch.complex64, (False, 64): torch.complex128}[(real, bits)]
    dev = D.device(dev)
    cv = (lambda M: D.to_cm(np.real(M) if real else M, dt, dev))
    tA, tB, tC = cv(A), cv(B), cv(C)
    npdt = {torch.float32: np.float32, torch.float64: np.float64, torch.complex64: np.complex64,
            torch.complex128: np.complex128}[dt]
    al = np.array([np.real(alpha) if real else alpha], dtype=npdt)
    be = np.array([np.real(beta) if real else beta], dtype=npdt)
    _native.check(_native.lib().sylv_gemm(D.dtype_code(tA), b"N", b"N", m, n, k, al.ctypes.data, tA.data_ptr(), m,
                                          tB.data_ptr(), k, be.ctypes.data, tC.data_ptr(), m, D.stream_ptr(dev)),
                  "sylv_gemm")
    return D.from_cm(tC).astype(np.complex128)
