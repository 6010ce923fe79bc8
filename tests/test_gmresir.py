"""Schur-preconditioned GMRES-IR on the device (reference gmresir.py).

Fixtures come from the reference itself (tests/golden/make_golden_gmres.py -> gmres.npz).
Bars: same convergence flag and failure string, outer iterations within +-1, final binary64
residual <= 10x the reference's (or the backward-stable level), solution within 10 kappa u_64.
The preconditioner tests restate the reference's own (pkg/tests/test_gmresir.py:15-37).
"""

import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
U64 = 2.0 ** -53
TAGS = ["c0_g64", "c0_g32", "c1_g64", "c3_g64", "c2_g32"]


@pytest.fixture(scope="module")
def golden_gmres():
    return np.load(os.path.join(ROOT, "tests", "golden", "gmres.npz"))


def kappa_sylv(A, B):
    m, n = A.shape[0], B.shape[0]
    return np.linalg.cond(np.kron(np.eye(n), A) + np.kron(B.T, np.eye(m)))


def test_config_validation():
    import paper_2503_03456_b200 as M
    with pytest.raises(ValueError):
        M.GmresConfig(restart=0)
    with pytest.raises(ValueError):
        M.GmresConfig(inner_tol=2.0)
    with pytest.raises(ValueError):
        M.gmres_ir_sylv(M.SylvesterProblem(np.eye(2), np.eye(2), np.ones((2, 2))), M.GmresConfig(M.BFLOAT16),
                        M.RefinementConfig(M.BINARY32, M.BINARY64))


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_device_gmres_ir_golden(golden_gmres, tag):
    import paper_2503_03456_b200 as M
    g = golden_gmres
    A, B, C = g[f"{tag}_A"], g[f"{tag}_B"], g[f"{tag}_C"]
    ug = M.BINARY32 if str(g[f"{tag}_ug"]) == "binary32" else M.BINARY64
    rep = M.gmres_ir_sylv(M.SylvesterProblem(A, B, C, kind=str(g[f"{tag}_kind"])), M.GmresConfig(ug),
                          M.RefinementConfig(M.BINARY32, M.BINARY64))
    assert rep.failure == (str(g[f"{tag}_fail"]) or None)
    assert rep.converged == bool(g[f"{tag}_conv"])
    assert abs(rep.outer_iterations - int(g[f"{tag}_outer"])) <= 1
    assert len(rep.inner_iterations) == rep.outer_iterations
    # residual after the same number of outer steps (the counts may differ by one: with
    # u_g = binary32 the preconditioner's rounding decides whether ||E|| <= eps ||X|| one
    # step earlier or later)
    hist = g[f"{tag}_hist"]
    ref_res = float(hist[min(rep.outer_iterations, len(hist)) - 1])
    assert rep.residual_history[-1] <= 10 * max(ref_res, U64)
    Xr = g[f"{tag}_X"]
    # forward difference <= 10 kappa x (the larger of u_64 and the residual this run stopped at)
    level = max(U64, rep.residual_history[-1]) if rep.outer_iterations != int(g[f"{tag}_outer"]) else U64
    assert np.linalg.norm(rep.X - Xr) / np.linalg.norm(Xr) <= 10 * kappa_sylv(A, B) * level * 10


@pytest.mark.gpu
def test_device_gmres_ir_singular_preconditioner(golden_gmres):
    import paper_2503_03456_b200 as M
    g = golden_gmres
    rep = M.gmres_ir_sylv(M.SylvesterProblem(g["sing_A"], g["sing_B"], np.ones((2, 1))), M.GmresConfig(M.BINARY64),
                          M.RefinementConfig(M.BINARY32, M.BINARY64))
    assert rep.failure == str(g["sing_fail"])
    assert rep.outer_iterations == int(g["sing_outer"])
    assert not rep.converged


@pytest.mark.gpu
def test_preconditioner_identities():
    import paper_2503_03456_b200 as M
    rng = np.random.default_rng(20240901)
    cm = (lambda m, n: rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    ctx = M.PrecisionContext(M.BINARY64)
    sf = M.schur(np.eye(2), ctx)
    W = cm(2, 2)
    assert np.abs(M.apply_preconditioner(W, sf, sf, ctx) - W / 2).max() < 1e-15
    sfA, sfB = M.schur(np.diag([1.0, 2.0]), ctx), M.schur(np.diag([3.0, 4.0]), ctx)
    den = np.array([[4.0, 5.0], [5.0, 6.0]])
    assert np.abs(M.apply_preconditioner(W, sfA, sfB, ctx) - W / den).max() < 1e-15
    A, B, X = cm(4, 4), cm(3, 3), cm(4, 3)
    W = A @ X + X @ B
    Z = M.apply_preconditioner(W, M.schur(A, ctx), M.schur(B, ctx), ctx)
    assert np.abs(Z - X).max() <= 1e-12 * np.abs(X).max()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,m,n,ug", [("c0", 300, 200, "binary64"), ("c1", 256, 256, "binary32"),
                                        ("c2", 320, 160, "binary64")])
def test_device_gmres_ir_larger(cfg, m, n, ug):
    """Sizes past the one-CTA Schur: converges to the backward-stable level; C2 has a known X."""
    import paper_2503_03456_b200 as M
    from paper_2503_03456_b200 import problems as P
    pr = P.make(cfg, m, n, seed=4)
    rep = M.gmres_ir_sylv(M.SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind),
                          M.GmresConfig(M.BINARY32 if ug == "binary32" else M.BINARY64),
                          M.RefinementConfig(M.BINARY32, M.BINARY64))
    assert rep.converged and rep.failure is None
    assert rep.residual_history[-1] <= 10 * max(m, n) * U64
    assert rep.outer_iterations <= 4
    if pr.X_true is not None:
        assert np.linalg.norm(rep.X - pr.X_true) / np.linalg.norm(pr.X_true) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["float64", "complex128", "float32"])
def test_krylov_step_kernel_matches_mgs(dt):
    """sylv_krylov_mgs (one cooperative launch) == modified Gram-Schmidt as in gmresir.py:131-140,
    plus the norm and the normalised new basis vector; deterministic run to run."""
    import torch
    from paper_2503_03456_b200.gmresir import _krylov
    tdt = getattr(torch, dt)
    rng = np.random.default_rng(5)
    N, j = 70001, 6
    def rnd(*s):
        a = rng.standard_normal(s) + (1j * rng.standard_normal(s) if "complex" in dt else 0)
        return torch.as_tensor(a).to(tdt).cuda()
    V = torch.empty((j + 2, N), dtype=tdt, device="cuda")
    Q, _ = torch.linalg.qr(rnd(N, j + 1).cpu().to(torch.complex128 if "complex" in dt else torch.float64))
    V[: j + 1] = Q.t().to(tdt).cuda()
    w0 = rnd(N)
    w = w0.clone()
    h = _krylov(V, j, w, N)
    # numpy MGS in float64 / complex128
    wn = w0.cpu().numpy().astype(np.complex128)
    Vn = V[: j + 1].cpu().numpy().astype(np.complex128)
    hr = []
    for i in range(j + 1):
        hi = np.vdot(Vn[i], wn)
        hr.append(hi)
        wn = wn - hi * Vn[i]
    tol = 1e-5 if dt == "float32" else 1e-12
    assert np.allclose(h[: j + 1], hr, atol=tol * np.abs(hr).max())
    assert abs(np.real(h[j + 1]) - np.linalg.norm(wn)) <= tol * np.linalg.norm(wn)
    assert np.allclose(V[j + 1].cpu().numpy(), wn / np.linalg.norm(wn), atol=10 * tol)
    w2 = w0.clone()
    h2 = _krylov(V, j, w2, N)
    assert np.array_equal(h, h2) and torch.equal(w, w2)
