"""Matrix-free condition number of the Sylvester operator, on the device.

The reference measures conditioning with kappa_2(M_f) of the explicit
Kronecker operator M_f = I_n (x) A + B^T (x) I_m (``cli.py:261-268``
``_condu``; ``linalg.py:656-707`` ``sylvester_kron_operator`` / ``sep_f``),
which it caps at mn <= DEFAULT_KRON_CAP.  At the BASELINE sizes (mn up to
1.7e7) M_f cannot be formed, so this module estimates the same quantity
without it:

  A = U_A T_A U_A^H, B = U_B T_B U_B^H (binary64 Schur, unitary U)
  =>  M_f = (conj(U_B) (x) U_A) M_T (conj(U_B) (x) U_A)^H,
      M_T Y = T_A Y + Y T_B, so M_f and M_T have the same singular values.

  sigma_min(M_T): inverse iteration on (M_T M_T^H)^{-1} -- each step one
      triangular Sylvester solve (sylv_trsyl) and one adjoint solve
      (T_A^H Z + Z T_B^H = W  <=>  T_B Z^H + Z^H T_A = W^H, sylv_trsyl again);
      the same iteration the reference's ``sep_f`` runs on the LU of M_f.
  sigma_max(M_T): power iteration on M_T^H M_T with sylv_gemm.

Both iterations converge from below, so kappa = sigma_max / sigma_min is a
lower bound that tightens with the iteration count (relative change <= rtol
between steps).  Everything runs through the C ABI on column-major device
tensors; torch only holds memory and takes vector norms.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from . import device as D
from .errors import SingularEquationError
from .linalg import schur_tensor
from .sylvester import _is_real, as_matrix


@dataclass(frozen=True)
class KappaEstimate:
    kappa: float
    sigma_max: float
    sigma_min: float
    iterations: tuple


def _scalar(dt, v):
    npdt = {torch.float64: np.float64, torch.complex128: np.complex128}[dt]
    return np.array([v], dtype=npdt)


def _gemm(opa, opb, A, B, C, alpha, beta, m, n, k, lda, ldb, ldc):
    dt = C.dtype
    al, be = _scalar(dt, alpha), _scalar(dt, beta)
    _native.check(_native.lib().sylv_gemm(D.dtype_code(C), opa, opb, m, n, k, al.ctypes.data, A.data_ptr(), lda,
                                          B.data_ptr(), ldb, be.ctypes.data, C.data_ptr(), ldc,
                                          D.stream_ptr(C.device)), "sylv_gemm")


def _trsyl(TA, TB, W, m, n):
    """In place: T_A Y + Y T_B = W (column-major tensors; W is (n, m) storage of m x n)."""
    L = _native.lib()
    code = D.dtype_code(W)
    sz = ct.c_size_t()
    _native.check(L.sylv_trsyl_workspace_size(code, m, n, ct.byref(sz)), "trsyl workspace")
    ws = D.workspace(sz.value, W.device)
    info = (ct.c_int * 4)()
    _native.check(L.sylv_trsyl(code, m, n, TA.data_ptr(), m, TB.data_ptr(), n, 0, W.data_ptr(), m, ws.data_ptr(),
                               sz.value, D.stream_ptr(W.device), info), "sylv_trsyl")
    if info[0] == _native.SINGULAR_EQUATION:
        raise SingularEquationError(info[1], info[2])
    return W


def _ct(W):
    """column-major conj-transpose: storage (c, r) of an r x c matrix -> storage (r, c) of its c x r adjoint."""
    return W.conj().t().contiguous() if W.is_complex() else W.t().contiguous()


def _start(m, n, dt, dev):
    v = torch.linspace(1.0, 2.0, m * n, dtype=torch.float64, device=dev).reshape(n, m).to(dt)
    return v / torch.linalg.vector_norm(v)


def sigma_min_triangular(TA, TB, m, n, max_iter=60, rtol=1e-4):
    """Smallest singular value of Y -> T_A Y + Y T_B (inverse iteration)."""
    v = _start(m, n, TA.dtype, TA.device)
    lam, it = 0.0, 0
    try:
        for it in range(1, max_iter + 1):
            z = _trsyl(TA, TB, v.clone(), m, n)               # M^{-1} v
            w = _ct(_trsyl(TB, TA, _ct(z), n, m))             # M^{-H} z
            lam_new = float(torch.linalg.vector_norm(w))
            if lam_new == 0.0 or not np.isfinite(lam_new):
                return 0.0, it
            v = w / lam_new
            done = abs(lam_new - lam) <= rtol * lam_new
            lam = lam_new
            if done:
                break
    except SingularEquationError:
        return 0.0, it
    return float(1.0 / np.sqrt(lam)), it


def sigma_max_triangular(TA, TB, m, n, max_iter=60, rtol=1e-4):
    """Largest singular value of Y -> T_A Y + Y T_B (power iteration on M^H M)."""
    v = _start(m, n, TA.dtype, TA.device)
    u = torch.empty_like(v)
    w = torch.empty_like(v)
    adj = b"C" if TA.is_complex() else b"T"
    lam, it = 0.0, 0
    for it in range(1, max_iter + 1):
        _gemm(b"N", b"N", TA, v, u, 1.0, 0.0, m, n, m, m, m, m)      # u = T_A v
        _gemm(b"N", b"N", v, TB, u, 1.0, 1.0, m, n, n, m, n, m)      # u += v T_B
        _gemm(adj, b"N", TA, u, w, 1.0, 0.0, m, n, m, m, m, m)       # w = T_A^H u
        _gemm(b"N", adj, u, TB, w, 1.0, 1.0, m, n, n, m, n, m)       # w += u T_B^H
        lam_new = float(torch.linalg.vector_norm(w))
        if lam_new == 0.0:
            return 0.0, it
        v = w / lam_new
        done = abs(lam_new - lam) <= rtol * lam_new
        lam = lam_new
        if done:
            break
    return float(np.sqrt(lam)), it


def kappa_sylv_tensor(A: torch.Tensor, B: torch.Tensor, max_iter=60, rtol=1e-4) -> KappaEstimate:
    """kappa_2 of M_f for column-major device tensors A (m x m) and B (n x n), float64 or complex128."""
    cx = A.is_complex() or B.is_complex()
    dt = torch.complex128 if cx else torch.float64
    TA, _ = schur_tensor(A.to(dt).clone())
    TB, _ = schur_tensor(B.to(dt).clone())
    m, n = TA.shape[0], TB.shape[0]
    smin, it1 = sigma_min_triangular(TA, TB, m, n, max_iter, rtol)
    smax, it2 = sigma_max_triangular(TA, TB, m, n, max_iter, rtol)
    kappa = float("inf") if smin == 0.0 else smax / smin
    return KappaEstimate(kappa, smax, smin, (it1, it2))


def kappa_sylv(A, B, max_iter=60, rtol=1e-4, dev=None) -> KappaEstimate:
    """kappa_2(I (x) A + B^T (x) I) for numpy A (m x m), B (n x n), estimated on the device."""
    A, B = as_matrix(A), as_matrix(B)
    real = _is_real(A, B)
    dt = torch.float64 if real else torch.complex128
    dev = D.device(dev)
    cv = (lambda M: D.to_cm(np.real(M) if real else M, dt, dev))
    return kappa_sylv_tensor(cv(A), cv(B), max_iter, rtol)
