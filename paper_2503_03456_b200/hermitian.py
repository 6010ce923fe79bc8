"""Hermitian fast path (drop-in for ``hermitian_eig`` linalg.py:583-640 and ``solve_hermitian``
sylvester.py:181-196).

For Hermitian A the unitary Schur form is diagonal, so the device Schur factorisation in
binary64 (``sylv_schur``: Hessenberg + multishift QR, unitary U to working accuracy) is the
eigendecomposition A = U diag(d) U^H with d = real(diag(T)); its strictly-upper part is at the
rounding level and is dropped.  This replaces the reference's cyclic complex Jacobi (the same
contract -- a unitary U and real d -- not the same iteration, so the eigenvalue order can
differ).  ``solve_hermitian`` then forms C~ = U_A^H C U_B and Y = C~ ./ (d_A + d_B^T) and
returns X = U_A Y U_B^H: two Schur factorisations, four GEMMs and one entrywise kernel
(``sylv_hdiv``), all through the C ABI.  binary64 only (the reference's default context).
"""

from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native
from . import device as D
from .condition import _gemm
from .errors import DimensionError, NotHermitianError, SingularEquationError, UnsupportedPrecisionError
from .linalg import schur_tensor
from .precision import format_bits
from .sylvester import as_matrix

_U64 = 2.0 ** -53


def _check_ctx(ctx):
    if ctx is not None and format_bits(getattr(ctx, "format", ctx)) != 64:
        raise UnsupportedPrecisionError("the device Hermitian path runs in binary64")


def _eig_tensor(A: torch.Tensor):
    """Column-major Hermitian device tensor -> (U, d) device tensors (U complex128, d float64).
    Always the complex Schur form: it is triangular (every 2x2 block split), so its diagonal
    is the spectrum even where a real quasi-triangular form would keep a 2x2 block."""
    T, U = schur_tensor(A.to(torch.complex128).clone())
    d = torch.diagonal(T).real.to(torch.float64).contiguous()
    return U, d


def hermitian_eig(A, ctx=None, dev=None):
    """A = U diag(d) U^H for Hermitian A (binary64); returns numpy (U complex128, d float64)."""
    _check_ctx(ctx)
    A = as_matrix(A)
    n = A.shape[0]
    if A.shape != (n, n):
        raise DimensionError("hermitian_eig requires a square matrix")
    nrm = float(np.linalg.norm(A))
    if float(np.linalg.norm(A - A.conj().T)) > 10 * _U64 * max(nrm, 1e-300):
        raise NotHermitianError("input is not Hermitian to working accuracy")
    if n == 1:
        return np.eye(1, dtype=np.complex128), np.array([A[0, 0].real])
    dev = D.device(dev)
    U, d = _eig_tensor(D.to_cm(A, torch.complex128, dev))
    return D.from_cm(U).astype(np.complex128), d.cpu().numpy()


def solve_hermitian(p, ctx=None, dev=None) -> np.ndarray:
    """X with A X + X B = C for Hermitian A, B (kind='hermitian'), binary64, on the device."""
    _check_ctx(ctx)
    if getattr(p, "kind", None) != "hermitian":
        raise ValueError("solve_hermitian requires kind='hermitian'")
    A, B, C = as_matrix(p.A), as_matrix(p.B), as_matrix(p.C)
    m, n = C.shape
    for M in (A, B):
        nrm = float(np.linalg.norm(M))
        if float(np.linalg.norm(M - M.conj().T)) > 10 * _U64 * max(nrm, 1e-300):
            raise NotHermitianError("input is not Hermitian to working accuracy")
    dt = torch.complex128  # the eigenvectors are complex (complex Schur); X is returned complex128
    dev = D.device(dev)
    cv = (lambda M: D.to_cm(M, dt, dev))
    tA, tB, tC = cv(A), cv(B), cv(C)
    if m > 1:
        UA, dA = _eig_tensor(tA)
    else:
        UA, dA = torch.ones((1, 1), dtype=dt, device=dev), tA.reshape(1).real.to(torch.float64)
    if n > 1:
        UB, dB = _eig_tensor(tB)
    else:
        UB, dB = torch.ones((1, 1), dtype=dt, device=dev), tB.reshape(1).real.to(torch.float64)
    adj = b"C"
    tmp = torch.empty_like(tC)
    Y = torch.empty_like(tC)
    _gemm(adj, b"N", UA, tC, tmp, 1.0, 0.0, m, n, m, m, m, m)     # U_A^H C
    _gemm(b"N", b"N", tmp, UB, Y, 1.0, 0.0, m, n, n, m, n, m)      # (U_A^H C) U_B
    L = _native.lib()
    ws = D.workspace(256, dev)
    info = (ct.c_int * 3)()
    _native.check(L.sylv_hdiv(D.dtype_code(Y), m, n, dA.data_ptr(), dB.data_ptr(), Y.data_ptr(), m, ws.data_ptr(),
                              256, D.stream_ptr(dev), info), "sylv_hdiv")
    if info[0] == _native.SINGULAR_EQUATION:
        raise SingularEquationError(info[1], info[2])
    _gemm(b"N", b"N", UA, Y, tmp, 1.0, 0.0, m, n, m, m, m, m)      # U_A Y
    X = torch.empty_like(tC)
    _gemm(b"N", adj, tmp, UB, X, 1.0, 0.0, m, n, n, m, n, m)       # (U_A Y) U_B^H
    return D.from_cm(X).astype(np.complex128)
