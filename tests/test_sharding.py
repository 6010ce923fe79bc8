"""Host-side logic of the batched (C4) path: shard boundaries, the batched
workspace query, and the one collective (final gather) on a world-size-2 gloo
group on CPU -- the same code the NCCL ranks run on the GPU box."""

import ctypes as ct
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_03456_b200.batch import gather_solutions, shard_range


@pytest.mark.parametrize("total,world", [(512, 1), (512, 2), (512, 8), (7, 3), (3, 8), (0, 2)])
def test_shard_range_partitions(total, world):
    spans = [shard_range(total, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_batched_workspace_query():
    from paper_2503_03456_b200 import _native
    L = _native.lib()
    p = _native.Params(m=512, n=512, kind=0, complex_data=0, variant=0, low_bits=32, correction_bits=64,
                       max_iter=20, y0_zero=0, epsilon=5.12e-10)
    one, many = ct.c_size_t(), ct.c_size_t()
    assert L.sylv_workspace_size(ct.byref(p), ct.byref(one)) == 0
    assert L.sylv_batched_workspace_size(ct.byref(p), 4, ct.byref(many)) == 0
    assert many.value >= 4 * one.value
    # an empty batch is a no-op and never touches the device
    reps = (_native.Report * 1)()
    assert L.sylv_solve_batched(ct.byref(p), 0, None, 512, None, 512, None, 512, None, 512, 4, None, 0, None,
                                reps) == 0
    assert L.sylv_solve_batched(ct.byref(p), -1, None, 512, None, 512, None, 512, None, 512, 4, None, 0, None,
                                reps) == _native.EINVAL


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(total, rank, world)
    # each rank "solves" its own equations: X[i] = i * ones (stand-in for the device result)
    X = torch.stack([torch.full((3, 2), float(i), dtype=torch.float64) for i in range(lo, hi)]) \
        if hi > lo else torch.zeros((0, 3, 2), dtype=torch.float64)
    out = gather_solutions(X, total)
    if rank == 0:
        q.put(out.numpy().copy())
    else:
        assert out is None
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 8])
def test_gather_solutions_gloo_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got.shape == (total, 3, 2)
    for i in range(total):
        assert (got[i] == i).all()


def _split_worker(rank, world, port, q):
    """The 2-GPU split's exchange (split2.exchange_b_factors) on gloo: rank 1 'factors' B (a
    stand-in for the device Schur) and sends (T_B, U_B) to rank 0; the other ranks idle."""
    from paper_2503_03456_b200.split2 import exchange_b_factors
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 5
    B = torch.arange(n * n, dtype=torch.float32).reshape(n, n) if rank == 1 else None
    got = exchange_b_factors(lambda Bm: (2 * Bm, Bm + 1), B, n, torch.float32, torch.device("cpu"), 0, 1)
    if rank == 0:
        q.put((got[0].numpy().copy(), got[1].numpy().copy()))
    else:
        assert got is None
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split2_exchange_gloo(world):
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    TB, UB = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    B = np.arange(25, dtype=np.float32).reshape(5, 5)
    assert np.array_equal(TB, 2 * B) and np.array_equal(UB, B + 1)
