"""Batched solves (config C4) and their multi-GPU sharding.

The reference solves independent equations one at a time through ``mp_orth`` /
``mp_inv`` (refinement.py:205-297); SPEC.md:369-370 allows independent solves to
run concurrently.  ``solve_batched`` hands a whole batch to the native lane
executor (``sylv_solve_batched``: concurrent lanes, one stream + host worker +
workspace slice each).  Across GPUs the batch shards by equation index with no
data-path collective; ``gather_solutions`` is the one exchange.
"""

from __future__ import annotations

import ctypes as ct

import torch

from . import _native
from . import device as D
from .errors import DeviceError, DimensionError


DEFAULT_LANES = 64  # kDefaultLanes in csrc/solver.cu


def effective_lanes(lanes: int, batch: int) -> int:
    """Lanes the executor actually runs: min(lanes or the default, batch), at least 1."""
    return max(1, min(lanes if lanes > 0 else DEFAULT_LANES, batch))


def _params(m, n, cx, kind, variant, low_bits, correction_bits, epsilon, max_iter, y0_zero):
    p = _native.Params()
    p.m, p.n = m, n
    p.kind = _native.KIND_LYAPUNOV if kind == "lyapunov" else _native.KIND_GENERAL
    p.complex_data = int(cx)
    p.variant = _native.VARIANT_INV if variant == "inv" else _native.VARIANT_ORTH
    p.low_bits, p.correction_bits = int(low_bits), int(correction_bits)
    p.max_iter, p.y0_zero, p.epsilon = int(max_iter), int(bool(y0_zero)), float(epsilon)
    return p


def solve_batched(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor, *, kind: str = "general",
                  variant: str = "orth", low_bits: int = 32, correction_bits: int = 64,
                  epsilon: float | None = None, max_iter: int = 20, y0_zero: bool = False,
                  lanes: int = 0, out: torch.Tensor | None = None):
    """Solve A[i] X[i] + X[i] B[i] = C[i] for every i.

    A (batch, m, m), B (batch, n, n), C (batch, m, n): row-major CUDA tensors
    (float64 -> real path, complex128 -> complex path).  Returns (X, reports):
    X (batch, m, n) and one native report per equation (``report.status``
    carries the typed failures, as in ``solve``).
    """
    if A.dim() != 3 or B.dim() != 3 or C.dim() != 3:
        raise DimensionError("expected (batch, rows, cols) tensors")
    nb, m, n = C.shape
    if A.shape != (nb, m, m) or B.shape != (nb, n, n):
        raise DimensionError(f"incompatible shapes A{tuple(A.shape)} B{tuple(B.shape)} C{tuple(C.shape)}")
    if not (A.is_cuda and B.is_cuda and C.is_cuda):
        raise DeviceError("solve_batched() expects CUDA tensors (no CPU fallback)")
    cx = A.is_complex() or B.is_complex() or C.is_complex()
    dt = torch.complex128 if cx else torch.float64
    A, B, C = (t.to(dt).contiguous() for t in (A, B, C))
    if out is None:
        out = torch.empty((nb, m, n), dtype=dt, device=A.device)
    if nb == 0:
        return out, []
    eps = epsilon if epsilon is not None else 1e-12 * max(m, n)
    # row-major storage == column-major transpose: solve B^T X^T + X^T A^T = C^T (order (n, m))
    p = _params(n, m, cx, kind, variant, low_bits, correction_bits, eps, max_iter, y0_zero)
    L = _native.lib()
    sz = ct.c_size_t()
    lanes = effective_lanes(int(lanes), nb)
    _native.check(L.sylv_batched_workspace_size(ct.byref(p), lanes, ct.byref(sz)), "workspace query")
    ws = D.workspace(sz.value, A.device)
    Arr = ct.c_void_p * nb
    es = A.element_size()
    pa = Arr(*[B.data_ptr() + i * n * n * es for i in range(nb)])
    pb = Arr(*[A.data_ptr() + i * m * m * es for i in range(nb)])
    pc = Arr(*[C.data_ptr() + i * m * n * es for i in range(nb)])
    px = Arr(*[out.data_ptr() + i * m * n * es for i in range(nb)])
    reps = (_native.Report * nb)()
    with torch.cuda.device(A.device):
        rc = L.sylv_solve_batched(ct.byref(p), nb, pa, n, pb, m, pc, n, px, n, int(lanes), ws.data_ptr(),
                                  sz.value, D.stream_ptr(A.device), reps)
    _native.check(rc, "sylv_solve_batched")
    return out, list(reps)


# ---- sharding across ranks (one process per GPU) -------------------------------------------

def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of equation indices [lo, hi) owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard request")
    q, r = divmod(total, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def gather_solutions(X_local: torch.Tensor, total: int, group=None):
    """Collect every rank's (count, m, n) block of solutions on rank 0, in equation order.

    The only collective of the batched path.  Blocks are padded to the largest shard so a single
    ``gather`` suffices (NCCL over NVLink on GPUs, gloo on CPU).  Returns the (total, m, n) tensor
    on rank 0 and None elsewhere.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    q = -(-total // world)
    pad = torch.zeros((q,) + tuple(X_local.shape[1:]), dtype=X_local.dtype, device=X_local.device)
    pad[: X_local.shape[0]] = X_local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    parts = []
    for r in range(world):
        lo, hi = shard_range(total, r, world)
        parts.append(bufs[r][: hi - lo])
    return torch.cat(parts, 0)
