"""Two-GPU task-parallel solve of ONE Sylvester equation (8e).

The only intra-solve split the algorithm offers: the two low-precision Schur
factorisations of Alg. 3/4 (``_low_precision_schur_pair``, refinement.py:190-197) are
independent.  Rank ``b_rank`` factors B while rank ``a_rank`` factors A; the B factors
(T_B, U_B: 2 n^2 low-precision words) are sent to the A rank, which finishes the solve with
``sylv_solve_factored`` (everything after the Schur pair is unchanged).  On one GPU the two
Schur factorisations share the SMs (the pair takes ~1.3x a single one at 4096); on two they
do not.  Lyapunov problems have one Schur and do not split.

    X, rep = mp_orth_split2(p, cfg)          # under torch.distributed with >= 2 ranks

The exchange is one point-to-point send (NCCL over NVLink on GPUs); the host logic is covered
with gloo on CPU (tests/test_sharding.py), the factored solve on one GPU
(tests/test_gpu_parity.py::test_factored_solve_matches_solve).
"""

from __future__ import annotations

import ctypes as ct

import numpy as np
import torch

from . import _native
from . import device as D
from .errors import DimensionError
from .linalg import schur_tensor
from .refinement import (SolveReport, _correction_bits, _failure_string, _precision_pair, _raise_for,
                         _resolve_eps)
from .sylvester import SylvesterProblem, _is_real

__all__ = ["exchange_b_factors", "solve_factored", "mp_orth_split2", "mp_inv_split2"]


def exchange_b_factors(factor_b, B_local, n, dtype, device, a_rank=0, b_rank=1, group=None):
    """Run ``factor_b(B_local) -> (T_B, U_B)`` on ``b_rank`` and deliver both factors to
    ``a_rank`` (one send of the stacked n x n pair).  Returns (T_B, U_B) on a_rank, None elsewhere."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if rank == b_rank:
        TB, UB = factor_b(B_local)
        dist.send(torch.stack([TB, UB]).contiguous(), dst=a_rank, group=group)
        return None
    if rank == a_rank:
        buf = torch.empty((2, n, n), dtype=dtype, device=device)
        dist.recv(buf, src=b_rank, group=group)
        return buf[0], buf[1]
    return None


def solve_factored(A, B, C, TA, UA, TB, UB, *, variant="orth", correction_bits=64, epsilon=None, max_iter=20,
                   y0_zero=False, kind="general"):
    """Column-major device tensors A (m x m), B (n x n), C (m x n) in high precision and the
    low-precision Schur factors (column-major): the solve after the Schur pair.  Returns
    (X column-major, native report)."""
    m, n = A.shape[0], B.shape[0]
    cx = A.is_complex()
    p = _native.Params()
    p.m, p.n = m, n
    p.kind = _native.KIND_LYAPUNOV if kind == "lyapunov" else _native.KIND_GENERAL
    p.complex_data = int(cx)
    p.variant = _native.VARIANT_INV if variant == "inv" else _native.VARIANT_ORTH
    p.low_bits = 32
    p.correction_bits = int(correction_bits)
    p.max_iter = int(max_iter)
    p.y0_zero = int(bool(y0_zero))
    p.epsilon = float(epsilon if epsilon is not None else 1e-12 * max(m, n))
    L = _native.lib()
    sz = ct.c_size_t()
    _native.check(L.sylv_workspace_size(ct.byref(p), ct.byref(sz)), "workspace query")
    ws = D.workspace(sz.value, A.device)
    X = torch.empty_like(C)
    rep = _native.Report()
    _native.check(L.sylv_solve_factored(ct.byref(p), A.data_ptr(), m, B.data_ptr(), n, C.data_ptr(), m,
                                        X.data_ptr(), m, TA.data_ptr(), m, UA.data_ptr(), m, TB.data_ptr(), n,
                                        UB.data_ptr(), n, ws.data_ptr(), sz.value, D.stream_ptr(A.device),
                                        ct.byref(rep)), "sylv_solve_factored")
    return X, rep


def _split2(p, cfg, variant, a_rank=0, b_rank=1, group=None):
    if not isinstance(p, SylvesterProblem):
        p = SylvesterProblem(p.A, p.B, p.C, kind=getattr(p, "kind", "general"))
    if p.kind == "lyapunov":
        raise DimensionError("a Lyapunov problem has one Schur factorisation: nothing to split")
    if _precision_pair(cfg) != 32:
        raise DimensionError("the split runs the (binary32, binary64) pair")
    import torch.distributed as dist
    rank = dist.get_rank(group)
    dev = D.device()
    m, n = p.m, p.n
    real = _is_real(p.A, p.B, p.C)
    dth = torch.float64 if real else torch.complex128
    dtl = torch.float32 if real else torch.complex64
    cv = (lambda M, dt: D.to_cm(np.real(M) if real else M, dt, dev))

    def factor(Bh):
        TB, UB = schur_tensor(cv(Bh, dtl))
        return TB, UB

    got = exchange_b_factors(factor, p.B if rank == b_rank else None, n, dtl, dev, a_rank, b_rank, group) \
        if rank in (a_rank, b_rank) else None
    if rank != a_rank:
        return None
    TA, UA = schur_tensor(cv(p.A, dtl))
    TB, UB = got
    tA, tB, tC = cv(p.A, dth), cv(p.B, dth), cv(p.C, dth)
    X, rep = solve_factored(tA, tB, tC, TA, UA, TB, UB, variant=variant, correction_bits=_correction_bits(cfg),
                            epsilon=_resolve_eps(cfg, m, n), max_iter=cfg.max_iter)
    _raise_for(rep.status)
    return SolveReport(D.from_cm(X).astype(np.complex128), int(rep.iterations), rep.norms(), float(rep.residual),
                       bool(rep.converged), _failure_string(rep), float(rep.backward_error))


def mp_orth_split2(p, cfg, a_rank=0, b_rank=1, group=None):
    """Alg. 3 (refinement.py:205-249) with Schur(A) on a_rank and Schur(B) on b_rank; the
    SolveReport is returned on a_rank (None on the others)."""
    return _split2(p, cfg, "orth", a_rank, b_rank, group)


def mp_inv_split2(p, cfg, a_rank=0, b_rank=1, group=None):
    """Alg. 4 (refinement.py:252-297) with the same split."""
    return _split2(p, cfg, "inv", a_rank, b_rank, group)
