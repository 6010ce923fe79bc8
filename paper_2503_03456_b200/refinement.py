"""Two-precision refinement solvers: the drop-in for ``mpsylv.refinement``.

Same entry points, arguments and results as the reference
(pkg/src/mpsylv/refinement.py): ``RefinementConfig`` (:47-75),
``SolveReport`` (:78-92), ``solve_pert_sylv_tri_stat`` (:95-141, Alg. 1),
``mp_orth`` (:205-249, Alg. 3) and ``mp_inv`` (:252-297, Alg. 4), with the
same typed failure strings.  All arithmetic runs in the sm_100a library
(``libmpsylv_b200.so``) through the C ABI; this module only validates,
moves data and rebuilds the report.

Precision pairs: (binary32, binary64) -> fp32/complex64 Schur + Y0 with
fp64/complex128 refinement; (binary64, binary64) -> everything in fp64.
Other pairs raise ``UnsupportedPrecisionError`` (the reference simulates
them in software; there is no simulator and no CPU fallback here).

Layout trick: a row-major m x n array is the column-major storage of its
transpose, and A X + X B = C  <=>  B^T X^T + X^T A^T = C^T.  The device is
handed (B, A, C) in row-major memory as the column-major problem
(A' = B^T, B' = A^T, C' = C^T), whose column-major solution X' = X^T is
exactly X in row-major memory: no transposes on either side.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from . import device as D
from .costmodel import algorithm_name, flops
from .errors import (DimensionError, FormatOverflowError, IterationLimitError, RankDeficiencyError,
                     SingularMatrixError, UnsupportedPrecisionError, DeviceError)
from .precision import BINARY64, FlopCounter, FpFormat, format_bits
from .sylvester import SylvesterProblem, _is_real

__all__ = ["RefinementConfig", "SolveReport", "solve", "solve_pert_sylv_tri_stat", "mp_orth", "mp_inv"]


@dataclass(frozen=True)
class RefinementConfig:
    """Precision pair and stopping rule (refinement.py:47-75)."""

    u_l: FpFormat = field(default_factory=lambda: BINARY64)
    u_h: FpFormat = field(default_factory=lambda: BINARY64)
    epsilon: float | None = None
    max_iter: int = 20
    # Opt-in extension (not in the reference): the precision of the correction solve
    # D_i = trsyl(T_A, T_B, R_i) inside Alg. 1.  None = u_h, the reference's choice
    # (refinement.py:124); BINARY32 = the north star's fast mode (R_i and the iterate stay
    # in binary64, only the triangular solve of the correction runs in binary32).
    correction: FpFormat | None = None

    def __post_init__(self):
        if self.u_h.unit_roundoff > self.u_l.unit_roundoff:
            raise ValueError("the high precision must not be coarser than the low one")
        if self.epsilon is not None and self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        if self.correction is not None and format_bits(self.correction) not in (32, 64):
            raise UnsupportedPrecisionError(
                f"correction precision {self.correction.name} is not computed natively on B200")

    def resolve_epsilon(self, m: int, n: int) -> float:
        if self.epsilon is not None:
            return self.epsilon
        if self.u_h.is_binary64:
            return 1e-12 * max(m, n)
        return 1e4 * self.u_h.unit_roundoff * max(m, n)


@dataclass(frozen=True)
class SolveReport:
    """Outcome of a refinement run (refinement.py:78-92) plus device diagnostics."""

    X: np.ndarray
    iterations: int
    correction_norms: list
    residual: float
    converged: bool
    failure: str | None = None
    backward_error: float = float("nan")
    timings_ms: dict = field(default_factory=dict, compare=False)


def _resolve_eps(cfg, m, n) -> float:
    if hasattr(cfg, "resolve_epsilon"):
        return float(cfg.resolve_epsilon(m, n))
    if cfg.epsilon is not None:
        return float(cfg.epsilon)
    return 1e-12 * max(m, n)


def _precision_pair(cfg):
    lo, hi = format_bits(cfg.u_l), format_bits(cfg.u_h)
    if hi != 64 or lo not in (32, 64):
        raise UnsupportedPrecisionError(
            f"precision pair ({cfg.u_l.name}, {cfg.u_h.name}) is not computed natively on B200; "
            "supported: (binary32, binary64), (binary64, binary64)")
    return lo


def _raise_for(status: int):
    if status == _native.FORMAT_OVERFLOW:
        raise FormatOverflowError("schur input has entries not representable in the low precision")
    if status == _native.ITERATION_LIMIT:
        raise IterationLimitError("QR iteration did not converge within its sweep budget")
    if status == _native.RANK_DEFICIENT:
        raise RankDeficiencyError("input is numerically rank deficient")
    if status == _native.SINGULAR_MATRIX:
        raise SingularMatrixError("exactly zero pivot in the LU factorization")


def _failure_string(rep: _native.Report):
    s = rep.status
    if s == _native.OK:
        return None
    pos = f"singular diagonal pair at position ({rep.fail_row}, {rep.fail_col})"
    if rep.fail_stage == _native.STAGE_INITIAL:
        if s == _native.SINGULAR_EQUATION:
            return f"singular_equation at initial triangular solve: {pos}"
        return f"nan_breakdown at initial triangular solve: non-finite values while solving column {rep.fail_col}"
    if s == _native.SINGULAR_EQUATION:
        return f"singular_equation during refinement: {pos}"
    if s == _native.NUMERIC_BREAKDOWN:
        if rep.fail_stage == _native.STAGE_DIVERGED:
            return "nan_breakdown: iterate diverged to non-finite values"
        return f"nan_breakdown: non-finite values while solving column {rep.fail_col}"
    if s == _native.NON_CONVERGENCE:
        return "non_convergence: correction ratio above epsilon at max_iter"
    return None


def solve(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor, *, kind: str = "general", variant: str = "orth",
          low_bits: int = 32, correction_bits: int = 64, epsilon: float | None = None, max_iter: int = 20,
          y0_zero: bool = False, out: torch.Tensor | None = None):
    """Torch-native entry: A (m x m), B (n x n), C (m x n) row-major device tensors.

    float64 tensors take the real path (fp32 Schur), complex128 the complex
    path (complex64 Schur).  variant: "orth" (mp_orth), "inv" (mp_inv) or "bs"
    (the fp64 Bartels-Stewart comparator: Schur in binary64, no refinement).  Returns (X, native report).  Raises the
    reference's exception types for raised errors; typed failures are in
    ``report.status`` (see ``_failure_string``).
    """
    if A.dim() != 2 or B.dim() != 2 or C.dim() != 2:
        raise DimensionError("expected 2-d matrices")
    m, n = C.shape
    if A.shape != (m, m) or B.shape != (n, n):
        raise DimensionError(f"incompatible shapes A{tuple(A.shape)} B{tuple(B.shape)} C{tuple(C.shape)}")
    if not (A.is_cuda and B.is_cuda and C.is_cuda):
        raise DeviceError("solve() expects CUDA tensors (no CPU fallback)")
    cx = A.is_complex() or B.is_complex() or C.is_complex()
    dt = torch.complex128 if cx else torch.float64
    A, B, C = (t.to(dt).contiguous() for t in (A, B, C))
    if out is None:
        out = torch.empty((m, n), dtype=dt, device=A.device)
    # column-major problem (A' = B^T, B' = A^T, C' = C^T) of order (n, m)
    if variant == "bs":
        low_bits = 64
    rep = _solve_cm(B, A, C, out, n, m, kind, variant, low_bits, correction_bits,
                    epsilon if epsilon is not None else 1e-12 * max(m, n), max_iter, y0_zero)
    return out, rep


def _solve_cm(A, B, C, X, m, n, kind, variant, low_bits, correction_bits, epsilon, max_iter, y0_zero):
    """Column-major call of sylv_solve: A (m x m), B (n x n), C and X (m x n), ld = rows."""
    p = _native.Params()
    p.m, p.n = m, n
    p.kind = _native.KIND_LYAPUNOV if kind == "lyapunov" else _native.KIND_GENERAL
    p.complex_data = int(A.is_complex())
    p.variant = {"inv": _native.VARIANT_INV, "bs": _native.VARIANT_BS}.get(variant, _native.VARIANT_ORTH)
    p.low_bits = int(low_bits)
    p.correction_bits = int(correction_bits)
    p.max_iter = int(max_iter)
    p.y0_zero = int(bool(y0_zero))
    p.epsilon = float(epsilon)
    L = _native.lib()
    sz = ct.c_size_t()
    _native.check(L.sylv_workspace_size(ct.byref(p), ct.byref(sz)), "workspace query")
    ws = D.workspace(sz.value, A.device)
    rep = _native.Report()
    with torch.cuda.device(A.device):
        rc = L.sylv_solve(ct.byref(p), A.data_ptr(), m, B.data_ptr(), n, C.data_ptr(), m, X.data_ptr(), m,
                          ws.data_ptr(), sz.value, D.stream_ptr(A.device), ct.byref(rep))
    _native.check(rc, "sylv_solve")
    return rep


def _correction_bits(cfg) -> int:
    c = getattr(cfg, "correction", None)
    return 64 if c is None else format_bits(c)


def _run(p, cfg, variant, counter, y0_zero):
    if not hasattr(p, "A"):
        raise TypeError("expected a SylvesterProblem")
    if not isinstance(p, SylvesterProblem):
        p = SylvesterProblem(p.A, p.B, p.C, kind=getattr(p, "kind", "general"))
    lo = _precision_pair(cfg)
    m, n = p.m, p.n
    eps = _resolve_eps(cfg, m, n)
    dev = D.device()
    real = _is_real(p.A, p.B, p.C)
    dt = torch.float64 if real else torch.complex128
    # same matrices as the reference (column-major copies, no transposed problem): Schur sees A and
    # B themselves, so structure the reference relies on (e.g. triangular inputs) is preserved
    cv = (lambda M: D.to_cm(np.real(M) if real else M, dt, dev))
    tA, tB, tC = cv(p.A), cv(p.B), cv(p.C)
    tX = torch.empty_like(tC)
    rep = _solve_cm(tA, tB, tC, tX, m, n, "lyapunov" if p.kind == "lyapunov" else "general", variant, lo,
                    _correction_bits(cfg), eps, cfg.max_iter, y0_zero)
    _raise_for(rep.status)
    Xn = D.from_cm(tX).astype(np.complex128)
    if counter is not None:  # model-derived counts (costmodel.flops), see precision.FlopCounter
        fc = flops(algorithm_name(variant, p.kind), m, n, rep.iterations)
        counter.add("low", int(round(fc.low_flops)))
        counter.add("high", int(round(fc.high_flops)))
    failure = _failure_string(rep)
    timings = dict(schur=rep.ms_schur, orth=rep.ms_orth, setup=rep.ms_setup, y0=rep.ms_y0,
                   refine=rep.ms_refine, recover=rep.ms_recover, total=rep.ms_total)
    return SolveReport(Xn, int(rep.iterations), rep.norms(), float(rep.residual), bool(rep.converged), failure,
                       float(rep.backward_error), timings)


def mp_orth(p, cfg: RefinementConfig, counter: FlopCounter | None = None, y0_zero: bool = False) -> SolveReport:
    """Alg. 3 (refinement.py:205-249): low-precision Schur, high-precision re-orthonormalisation."""
    return _run(p, cfg, "orth", counter, y0_zero)


def mp_inv(p, cfg: RefinementConfig, counter: FlopCounter | None = None, y0_zero: bool = False) -> SolveReport:
    """Alg. 4 (refinement.py:252-297): low-precision Schur, LU-based inverses in high precision."""
    return _run(p, cfg, "inv", counter, y0_zero)


def solve_pert_sylv_tri_stat(T_A, dT_A, T_B, dT_B, C, Y0, cfg: RefinementConfig,
                             counter: FlopCounter | None = None) -> SolveReport:
    """Alg. 1 (refinement.py:95-141): stationary refinement of the perturbed triangular equation."""
    from .sylvester import _triangular_form, as_matrix
    if format_bits(cfg.u_h) != 64:
        raise UnsupportedPrecisionError("the refinement runs in binary64")
    T_A, dT_A, T_B, dT_B, C, Y0 = (as_matrix(M) for M in (T_A, dT_A, T_B, dT_B, C, Y0))
    m, n = C.shape
    real = _is_real(T_A, dT_A, T_B, dT_B, C, Y0)
    if _triangular_form(T_A, real) != "upper":
        raise DimensionError("T_A must be upper triangular")
    lower = n > 1 and _triangular_form(T_B, real) == "lower"
    dev = D.device()
    dt = torch.float64 if real else torch.complex128
    cv = (lambda M: D.to_cm(np.real(M) if real else M, dt, dev))
    tTA, tdA, tTB, tdB, tC, tY0 = (cv(M) for M in (T_A, dT_A, T_B, dT_B, C, Y0))
    tY = torch.empty_like(tY0)
    code = 1 if real else 3
    L = _native.lib()
    sz = ct.c_size_t()
    _native.check(L.sylv_refine_workspace_size(code, m, n, ct.byref(sz)), "refine workspace")
    ws = D.workspace(sz.value, dev)
    rep = _native.Report()
    rc = L.sylv_refine(code, m, n, tTA.data_ptr(), m, tdA.data_ptr(), m, tTB.data_ptr(), n, tdB.data_ptr(), n,
                       int(lower), tC.data_ptr(), m, tY0.data_ptr(), m, float(_resolve_eps(cfg, m, n)),
                       int(cfg.max_iter), tY.data_ptr(), m, ws.data_ptr(), sz.value, D.stream_ptr(dev),
                       ct.byref(rep))
    _native.check(rc, "sylv_refine")
    if rep.status == _native.SINGULAR_EQUATION:
        from .errors import SingularEquationError
        raise SingularEquationError(rep.fail_row, rep.fail_col)
    failure = _failure_string(rep)
    return SolveReport(D.from_cm(tY).astype(np.complex128), int(rep.iterations), rep.norms(),
                       float(rep.residual), bool(rep.converged), failure)
