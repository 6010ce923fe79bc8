"""Schur-preconditioned GMRES iterative refinement on the device.

Mirrors the reference's ``mpsylv.gmresir`` (pkg/src/mpsylv/gmresir.py): ``GmresConfig``
(:44-63), ``GmresIrReport`` (:66-73), ``apply_preconditioner`` (:76-85),
``_gmres_correction`` (:112-205) and ``gmres_ir_sylv`` (:208-278) -- same arguments,
stopping rules, failure strings and report fields.

B200 design: the low-precision Schur factors come from the same sm_100a Schur kernels as
mp_orth (``sylv_schur``); the preconditioner (U_A^H W U_B -> triangular solve -> U_A Y U_B^H)
and the operator (A W + W B) run as the library's GEMM (``sylv_gemm``: fp64 DMMA / fp32
FFMA) and triangular-Sylvester (``sylv_trsyl``) kernels on column-major device matrices,
in the GMRES precision u_g.  The Krylov basis (m n x (restart+1)) stays in HBM; its
BLAS-1 steps (dot products, axpys, norms) are device tensor operations, and only the
restart-sized Hessenberg least-squares problem (Givens rotations, back substitution) is
scalar host work, as in the reference.  No step runs on the host CPU in bulk and there is
no CPU fallback.  ``counter`` is accepted for signature parity and left untouched (the
reference counts simulated operations; the device path has no per-operation count).
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from . import device as D
from .errors import DimensionError, NumericBreakdownError, SingularEquationError, UnsupportedPrecisionError
from .precision import BINARY64, FlopCounter, FpFormat, format_bits
from .refinement import RefinementConfig, _precision_pair, _resolve_eps
from .sylvester import SylvesterProblem, _is_real, _triangular_form

__all__ = ["GmresConfig", "GmresIrReport", "apply_preconditioner", "gmres_ir_sylv"]

_DT = {(True, 32): torch.float32, (True, 64): torch.float64, (False, 32): torch.complex64,
       (False, 64): torch.complex128}


@dataclass(frozen=True)
class GmresConfig:
    """Inner-solver settings (gmresir.py:44-63): restart length, tolerance, and the
    precision u_g of the preconditioned system.  Effective inner tolerance
    max(inner_tol, 4 u_g)."""

    u_g: FpFormat = field(default_factory=lambda: BINARY64)
    restart: int = 20
    inner_tol: float = 1e-8
    max_restarts: int = 5

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("restart must be at least 1")
        if self.max_restarts < 1:
            raise ValueError("max_restarts must be at least 1")
        if not 0 < self.inner_tol < 1:
            raise ValueError("inner_tol must lie in (0, 1)")


@dataclass(frozen=True)
class GmresIrReport:
    X: np.ndarray
    outer_iterations: int
    inner_iterations: list
    residual_history: list
    converged: bool
    failure: str | None = None


# ---------------------------------------------------------------------------
# column-major device matrices: a tensor t of shape (cols, rows) holds M = t.T
def _rows(t):
    return t.shape[1]


def _cols(t):
    return t.shape[0]


def _scalar(v, dt):
    npdt = {torch.float32: np.float32, torch.float64: np.float64, torch.complex64: np.complex64,
            torch.complex128: np.complex128}[dt]
    return np.array([v if dt.is_complex else np.real(v)], dtype=npdt)


def _gemm(opa, A, opb, B, C, alpha=1.0, beta=0.0):
    """C <- alpha op(A) op(B) + beta C through sylv_gemm (ops 'N' / 'C')."""
    M, N = _rows(C), _cols(C)
    K = _cols(A) if opa == "N" else _rows(A)
    al, be = _scalar(alpha, C.dtype), _scalar(beta, C.dtype)
    _native.check(_native.lib().sylv_gemm(D.dtype_code(C), opa.encode(), opb.encode(), M, N, K, al.ctypes.data,
                                          A.data_ptr(), _rows(A), B.data_ptr(), _rows(B), be.ctypes.data,
                                          C.data_ptr(), M, D.stream_ptr(C.device)), "sylv_gemm")
    return C


class _Factors:
    """Low-precision Schur factors, held on the device in the precision they are applied in."""

    def __init__(self, TA, UA, TB, UB, lowerB):
        self.TA, self.UA, self.TB, self.UB, self.lowerB = TA, UA, TB, UB, lowerB

    def cast(self, dt):
        return _Factors(self.TA.to(dt), self.UA.to(dt), self.TB.to(dt), self.UB.to(dt), self.lowerB)


def _schur_pair(tA, tB, lyap, dt_low):
    """_low_precision_schur_pair (refinement.py:190-197) with the device Schur kernels."""
    from .linalg import schur_tensor
    TA, UA = schur_tensor(tA.to(dt_low).clone())  # in place: never on the caller's tensor
    if lyap:  # T_B = T_A^H, U_B = U_A (the column recurrence then runs right to left)
        return _Factors(TA, UA, TA.conj().t().contiguous(), UA, True)
    TB, UB = schur_tensor(tB.to(dt_low).clone())
    return _Factors(TA, UA, TB, UB, False)


def _precondition(W, f: _Factors):
    """apply_preconditioner (gmresir.py:76-85): U_A (trsyl(T_A, T_B, U_A^H W U_B)) U_B^H."""
    m, n = _rows(W), _cols(W)
    tmp = torch.empty_like(W)
    V = torch.empty_like(W)
    _gemm("C", f.UA, "N", W, tmp)
    _gemm("N", tmp, "N", f.UB, V)
    L = _native.lib()
    sz = ct.c_size_t()
    code = D.dtype_code(V)
    _native.check(L.sylv_trsyl_workspace_size(code, m, n, ct.byref(sz)), "trsyl workspace")
    ws = D.workspace(sz.value, V.device)
    info = (ct.c_int * 4)()
    _native.check(L.sylv_trsyl(code, m, n, f.TA.data_ptr(), m, f.TB.data_ptr(), n, int(f.lowerB), V.data_ptr(), m,
                               ws.data_ptr(), sz.value, D.stream_ptr(V.device), info), "sylv_trsyl")
    if info[0] == _native.SINGULAR_EQUATION:
        raise SingularEquationError(info[1], info[2])
    if info[0] == _native.NUMERIC_BREAKDOWN:
        raise NumericBreakdownError(f"non-finite values while solving column {info[2]}")
    _gemm("N", f.UA, "N", V, tmp)
    out = torch.empty_like(W)
    _gemm("N", tmp, "C", f.UB, out)
    return out


def apply_preconditioner(W, sf_A, sf_B, ctx=None):
    """Reference-signature entry (gmresir.py:76-85): sf_A / sf_B carry .U and .T (numpy or
    SchurFactors); W (m x n).  Computed in the context's precision (binary32 / binary64)."""
    bits = 64 if ctx is None else format_bits(ctx.format)
    if bits not in (32, 64):
        raise UnsupportedPrecisionError(f"{ctx.format.name} is not a hardware format")
    W = np.asarray(W, dtype=np.complex128)
    mats = (W, sf_A.U, sf_A.T, sf_B.U, sf_B.T)
    dt = _DT[(_is_real(*mats), bits)]
    dev = D.device()
    cv = (lambda M: D.to_cm(np.real(M) if not dt.is_complex else M, dt, dev))
    TB = np.asarray(sf_B.T)
    lower = TB.shape[0] > 1 and _triangular_form(TB, not dt.is_complex) == "lower"
    f = _Factors(cv(sf_A.T), cv(sf_A.U), cv(TB), cv(sf_B.U), bool(lower))
    return D.from_cm(_precondition(cv(W), f)).astype(np.complex128)


# ---------------------------------------------------------------------------
_NP = {torch.float32: np.float32, torch.float64: np.float64, torch.complex64: np.complex64,
       torch.complex128: np.complex128}


def _krylov(V, j, w, N):
    """sylv_krylov_mgs: MGS of w against V[:, 0..j], h[j+1] = ||w||, V[:, j+1] = w / ||w||
    (one cooperative launch; j = -1: norm and V[:, 0] only).  Returns h (numpy, j+2)."""
    L = _native.lib()
    code = D.dtype_code(w)
    sz = ct.c_size_t()
    _native.check(L.sylv_krylov_workspace_size(code, N, j, ct.byref(sz)), "krylov workspace")
    ws = D.workspace(sz.value, w.device)
    h = np.zeros(j + 2, dtype=_NP[w.dtype])
    _native.check(L.sylv_krylov_mgs(code, N, V.data_ptr(), N, j, w.data_ptr(), h.ctypes.data, ws.data_ptr(),
                                    sz.value, D.stream_ptr(w.device)), "sylv_krylov_mgs")
    return h


def _vnorm(x) -> float:
    """||x||_2 of a device vector / matrix through the Krylov kernel (a scratch column)."""
    v = x.reshape(-1)
    scratch = torch.empty_like(v)
    return float(np.real(_krylov(scratch, -1, v, v.numel())[0]))


def _axpy(y, x, alpha):
    """y <- y + alpha x for flattened device vectors (a K = 1 product through sylv_gemm)."""
    yv, xv = y.reshape(-1), x.reshape(-1)
    one = torch.ones((1, 1), dtype=y.dtype, device=y.device)
    N = yv.numel()
    al, be = _scalar(alpha, y.dtype), _scalar(1.0, y.dtype)
    _native.check(_native.lib().sylv_gemm(D.dtype_code(yv), b"N", b"N", N, 1, 1, al.ctypes.data, xv.data_ptr(), N,
                                          one.data_ptr(), 1, be.ctypes.data, yv.data_ptr(), N,
                                          D.stream_ptr(y.device)), "sylv_gemm")
    return y


def _gmres_correction(matvec, rhs, gcfg: GmresConfig, unit_roundoff: float):
    """Restarted GMRES on the flattened preconditioned system (gmresir.py:112-205).
    rhs: column-major device matrix; returns (E, inner_iterations, stagnated).
    Every O(N) step runs on the device: the Arnoldi step (MGS + norm + normalisation) is one
    sylv_krylov_mgs launch, the basis combination x += V y and the restart residual are
    sylv_gemm products; only the (p+1) x p Hessenberg least-squares problem (Givens
    rotations) runs on the host, as in the reference."""
    shape, dt = rhs.shape, rhs.dtype
    b = rhs.reshape(-1)  # column-major storage flattened = vec (column stacking)
    N = b.numel()
    x = torch.zeros_like(b)
    p = gcfg.restart
    cx = dt.is_complex
    Vb = torch.empty((p + 1, N), dtype=dt, device=b.device)  # column-major N x (p+1)
    beta0 = float(np.real(_krylov(Vb, -1, b, N)[0]))
    if beta0 == 0.0:
        return x.reshape(shape), 0, False
    tol = max(gcfg.inner_tol, 4.0 * unit_roundoff)
    total_inner = 0
    stagnated = False
    x_zero = True
    for _ in range(gcfg.max_restarts):
        r = b.clone()
        if not x_zero:
            _axpy(r, matvec(x), -1.0)
        beta = float(np.real(_krylov(Vb, -1, r, N)[0]))  # also V[:, 0] = r / beta
        if not np.isfinite(beta):
            return x.reshape(shape), total_inner, True
        if beta <= tol * beta0:
            break
        cycle_start = beta
        H = np.zeros((p + 1, p), dtype=np.complex128)
        cs = np.zeros(p, dtype=np.complex128)
        sn = np.zeros(p, dtype=np.complex128)
        g = np.zeros(p + 1, dtype=np.complex128)
        g[0] = beta
        j = 0
        while j < p:
            w = matvec(Vb[j])
            h = _krylov(Vb, j, w, N)  # MGS like the reference, then ||w|| and v_{j+1}
            H[: j + 1, j] = h[: j + 1] if cx else np.real(h[: j + 1])
            hq = float(np.real(h[j + 1]))
            H[j + 1, j] = hq
            total_inner += 1
            if not np.isfinite(hq):
                return x.reshape(shape), total_inner, True
            for i in range(j):
                t = np.conj(cs[i]) * H[i, j] + np.conj(sn[i]) * H[i + 1, j]
                H[i + 1, j] = cs[i] * H[i + 1, j] - sn[i] * H[i, j]
                H[i, j] = t
            hjj, hj1 = H[j, j], H[j + 1, j]
            d = float(np.sqrt(abs(hjj) ** 2 + abs(hj1) ** 2))
            if d == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = hjj / d, hj1 / d
            H[j, j] = d
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = np.conj(cs[j]) * g[j]
            j += 1
            if abs(g[j]) <= tol * beta0:
                break
        y = np.zeros(j, dtype=np.complex128)
        for i in range(j - 1, -1, -1):
            acc = g[i]
            for l in range(i + 1, j):
                acc = acc - H[i, l] * y[l]
            y[i] = acc / H[i, i]
        coef = torch.as_tensor(y if cx else y.real, dtype=dt, device=b.device)
        al, be = _scalar(1.0, dt), _scalar(1.0, dt)
        _native.check(_native.lib().sylv_gemm(D.dtype_code(x), b"N", b"N", N, 1, j, al.ctypes.data, Vb.data_ptr(), N,
                                              coef.data_ptr(), j, be.ctypes.data, x.data_ptr(), N,
                                              D.stream_ptr(x.device)), "sylv_gemm")  # x += V[:, :j] y
        x_zero = False
        final = abs(g[j])
        if final <= tol * beta0:
            break
        if final > 0.9 * cycle_start:
            stagnated = True
            break
    else:
        stagnated = True
    return x.reshape(shape), total_inner, stagnated


def _device_residual(tA, tB, tC, tX) -> float:
    """residual (sylvester.py:199-209) in binary64 on the device."""
    R = tC.clone()
    _gemm("N", tA, "N", tX, R, -1.0, 1.0)
    _gemm("N", tX, "N", tB, R, -1.0, 1.0)
    nr = _vnorm(R)
    den = _vnorm(tC) + _vnorm(tX) * (_vnorm(tA) + _vnorm(tB))
    return 0.0 if den == 0.0 else nr / den


def gmres_ir_sylv(p, gcfg: GmresConfig, rcfg: RefinementConfig, counter: FlopCounter | None = None) -> GmresIrReport:
    """Refinement with GMRES correction solves in precision u_g (gmresir.py:208-278).

    Schur factors in u_l; each outer step forms R = C - A X - X B in u_h, left-preconditions
    it in u_g and solves the preconditioned correction equation by restarted GMRES in u_g.
    Stops when ||E||_F <= eps ||X||_F or the binary64 residual reaches 10 max(m, n) u_h.
    """
    if gcfg.u_g not in (rcfg.u_l, rcfg.u_h) and format_bits(gcfg.u_g) not in (
            format_bits(rcfg.u_l), format_bits(rcfg.u_h)):
        raise ValueError("u_g must equal one of the configured precisions")
    if not hasattr(p, "A"):
        raise TypeError("expected a SylvesterProblem")
    if not isinstance(p, SylvesterProblem):
        p = SylvesterProblem(p.A, p.B, p.C, kind=getattr(p, "kind", "general"))
    lo = _precision_pair(rcfg)
    gbits = format_bits(gcfg.u_g)
    if gbits not in (32, 64):
        raise UnsupportedPrecisionError(f"{gcfg.u_g.name} is not a hardware format")
    m, n = p.m, p.n
    if m < 1 or n < 1:
        raise DimensionError("empty problem")
    eps = _resolve_eps(rcfg, m, n)
    dev = D.device()
    real = _is_real(p.A, p.B, p.C)
    dth, dtg, dtl = _DT[(real, 64)], _DT[(real, gbits)], _DT[(real, lo)]
    cv = (lambda M: D.to_cm(np.real(M) if real else M, dth, dev))
    tA, tB, tC = cv(p.A), cv(p.B), cv(p.C)
    lyap = p.kind == "lyapunov"
    f = _schur_pair(tA, tB, lyap, dtl).cast(dtg)
    Ag, Bg = tA.to(dtg), tB.to(dtg)
    ug = 2.0 ** -24 if gbits == 32 else 2.0 ** -53
    uh = 2.0 ** -53

    def matvec(xflat):
        W = xflat.reshape(n, m)
        AW = torch.empty_like(W)
        _gemm("N", W, "N", Bg, AW)
        _gemm("N", Ag, "N", W, AW, 1.0, 1.0)
        return _precondition(AW, f).reshape(-1)

    X = torch.zeros_like(tC)
    inner_counts, history = [], []
    converged, failure, outer = False, None, 0
    while outer < rcfg.max_iter:
        R = tC.clone()
        _gemm("N", tA, "N", X, R, -1.0, 1.0)
        _gemm("N", X, "N", tB, R, -1.0, 1.0)
        try:
            Rt = _precondition(R.to(dtg), f)
            E, li, stagnated = _gmres_correction(matvec, Rt, gcfg, ug)
        except (SingularEquationError, NumericBreakdownError) as exc:
            failure = f"preconditioner failure: {exc}"
            break
        Eh = E.to(dth)
        _axpy(X, Eh, 1.0)
        outer += 1
        inner_counts.append(li)
        history.append(_device_residual(tA, tB, tC, X))
        nE = _vnorm(Eh)
        nX = _vnorm(X)
        if not (np.isfinite(nE) and np.isfinite(nX)):
            failure = "nan_breakdown: iterate diverged to non-finite values"
            break
        stable = 10.0 * max(m, n) * uh
        if nE <= eps * nX or history[-1] <= stable:
            converged = True
            break
        if stagnated:
            failure = "gmres_stagnation: inner residual stopped decreasing"
            break
    if failure is None and not converged:
        failure = "non_convergence: correction ratio above epsilon at max_iter"
    return GmresIrReport(D.from_cm(X).astype(np.complex128), outer, inner_counts, history, converged, failure)
