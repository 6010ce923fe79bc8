"""The fp64 Bartels-Stewart comparator (reference sylvester.py:160-178).

CPU: the oracle's composition (oracle.bartels_stewart) against the reference's own
outputs (tests/golden/make_golden_bs.py -> bs.npz).  GPU: the device path
(sylv_solve with SYLV_VARIANT_BS, Schur in binary64) against the same fixtures and
against the oracle on seeded inputs at larger sizes; the bar is the north star's
(backward error <= 10x the reference's, solution within 10 kappa u_64).
"""

import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
U64 = 2.0 ** -53
TAGS = ["c0", "c1", "c2", "c3"]


@pytest.fixture(scope="module")
def golden_bs():
    return np.load(os.path.join(ROOT, "tests", "golden", "bs.npz"))


def backward(A, B, C, X):
    return np.linalg.norm(A @ X + X @ B - C) / ((np.linalg.norm(A) + np.linalg.norm(B)) * np.linalg.norm(X))


def kappa_sylv(A, B):
    m, n = A.shape[0], B.shape[0]
    return np.linalg.cond(np.kron(np.eye(n), A) + np.kron(B.T, np.eye(m)))


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_bs_matches_reference(oracle, golden_bs, tag):
    g = golden_bs
    A, B, C = g[f"{tag}_A"], g[f"{tag}_B"], g[f"{tag}_C"]
    X, res = oracle.bartels_stewart(A, B, C, kind=str(g[f"{tag}_kind"]))
    Xr = g[f"{tag}_X"]
    # binary64 throughout: agreement to a few ulps scaled by the conditioning
    assert np.linalg.norm(X - Xr) / np.linalg.norm(Xr) <= 100 * kappa_sylv(A, B) * U64
    assert abs(res - float(g[f"{tag}_res"])) <= 1e-15


def test_oracle_bs_singular(oracle, golden_bs):
    g = golden_bs
    with pytest.raises(oracle.OracleError) as e:
        oracle.bartels_stewart(g["sing_A"], g["sing_B"], np.ones((2, 1)))
    assert (e.value.row, e.value.col) == tuple(int(v) for v in g["sing_rowcol"])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_device_bs_golden(golden_bs, tag):
    import paper_2503_03456_b200 as M
    g = golden_bs
    A, B, C = g[f"{tag}_A"], g[f"{tag}_B"], g[f"{tag}_C"]
    X, rep = M.bartels_stewart(M.SylvesterProblem(A, B, C, kind=str(g[f"{tag}_kind"])))
    Xr = g[f"{tag}_X"]
    assert backward(A, B, C, X) <= 10 * max(backward(A, B, C, Xr), U64)
    assert np.linalg.norm(X - Xr) / np.linalg.norm(Xr) <= 10 * kappa_sylv(A, B) * U64
    assert rep.residual <= 10 * max(float(g[f"{tag}_res"]), U64)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,m,n", [("c0", 150, 96), ("c1", 140, 140), ("c2", 160, 80), ("c3", 100, 72)])
def test_device_bs_vs_oracle(oracle, cfg, m, n):
    import paper_2503_03456_b200 as M
    from paper_2503_03456_b200 import problems as P
    pr = P.make(cfg, m, n, seed=11)
    X, rep = M.bartels_stewart(M.SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind))
    Xo, _ = oracle.bartels_stewart(pr.A, pr.B, pr.C, kind=pr.kind)
    A, B, C = pr.A, pr.B, pr.C
    assert backward(A, B, C, X) <= 10 * max(backward(A, B, C, Xo), U64)
    kap = kappa_sylv(A, B) if m * n <= 4096 else 10.0  # recipes have kappa ~3-10
    assert np.linalg.norm(X - Xo) / np.linalg.norm(Xo) <= 10 * kap * U64 * 10
    if pr.kind == "lyapunov":
        assert np.linalg.norm(X - X.conj().T) / np.linalg.norm(X) <= 1e-13


@pytest.mark.gpu
def test_device_bs_singular_raises(golden_bs):
    import paper_2503_03456_b200 as M
    g = golden_bs
    with pytest.raises(M.SingularEquationError) as e:
        M.bartels_stewart(M.SylvesterProblem(g["sing_A"], g["sing_B"], np.ones((2, 1))))
    assert (e.value.row, e.value.col) == tuple(int(v) for v in g["sing_rowcol"])


@pytest.mark.gpu
def test_device_bs_torch_api_and_known_solution():
    import torch
    import paper_2503_03456_b200 as M
    from paper_2503_03456_b200 import problems as P
    pr = P.make("c2", 384, 256, seed=5)  # known X_true
    dev = torch.device("cuda", 0)
    A, B, C = (torch.as_tensor(x, device=dev) for x in (pr.A, pr.B, pr.C))
    X, rep = M.solve(A, B, C, variant="bs")
    assert rep.status == 0 and rep.iterations == 0
    fwd = np.linalg.norm(X.cpu().numpy() - pr.X_true) / np.linalg.norm(pr.X_true)
    assert fwd <= 1e-12, fwd
    assert rep.backward_error <= 1e-15


def test_bs_precision_guard():
    import paper_2503_03456_b200 as M
    with pytest.raises(M.UnsupportedPrecisionError):
        M.bartels_stewart(M.SylvesterProblem(np.eye(2), np.eye(2), np.ones((2, 2))),
                          M.PrecisionContext(M.BINARY32))
