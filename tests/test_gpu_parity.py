"""End-to-end parity of mp_orth / mp_inv on the B200 against the reference.

Bars (BASELINE.json north star): refinement iterations within +-1 of the
reference's, normwise backward error ||C-AX-XB||_F/((||A||_F+||B||_F)||X||_F)
at most 10x the reference's, relative solution difference within
10 * kappa_sylv * u_fp64 (kappa_sylv = kappa_2 of the Kronecker operator,
the reference's own convention, cli.py:261-268, computed where mn <= 4096).

Reference answers come from (a) the committed golden fixtures produced by the
Python reference itself and (b) the bit-exact CPU oracle on the same seeded
inputs at sizes it finishes in seconds.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U64 = 2.0 ** -53


@pytest.fixture(scope="module")
def B200():
    import torch
    assert torch.cuda.is_available()
    import paper_2503_03456_b200 as M
    return M


def backward(A, B, C, X):
    return np.linalg.norm(A @ X + X @ B - C) / ((np.linalg.norm(A) + np.linalg.norm(B)) * np.linalg.norm(X))


def kappa_sylv(A, B):
    m, n = A.shape[0], B.shape[0]
    M = np.kron(np.eye(n), A) + np.kron(B.T, np.eye(m))
    return np.linalg.cond(M)


def cfg_for(M, ul):
    return M.RefinementConfig(M.BINARY32 if ul == "binary32" else M.BINARY64, M.BINARY64)


def check_parity(rep, X_ref, k_ref, A, B, C, kappa=None, kslack=1):
    assert rep.failure is None, rep.failure
    assert abs(rep.iterations - k_ref) <= kslack, (rep.iterations, k_ref)
    be_ref = backward(A, B, C, X_ref)
    be = backward(A, B, C, rep.X)
    assert be <= 10 * max(be_ref, U64), (be, be_ref)
    if kappa is not None:
        fwd = np.linalg.norm(rep.X - X_ref) / np.linalg.norm(X_ref)
        assert fwd <= 10 * kappa * U64, (fwd, kappa)


def _tags(s):
    return sorted({key.rsplit("_", 1)[0] for key in s.files if key.endswith("_kind")})


@pytest.mark.parametrize("variant", ["orth", "inv"])
def test_golden_fixtures(B200, golden_solves, variant):
    s = golden_solves
    for t in _tags(s):
        A, B, C = s[f"{t}_A"], s[f"{t}_B"], s[f"{t}_C"]
        p = B200.SylvesterProblem(A, B, C, kind=str(s[f"{t}_kind"]))
        solver = B200.mp_orth if variant == "orth" else B200.mp_inv
        rep = solver(p, cfg_for(B200, str(s[f"{t}_ul"])))
        check_parity(rep, s[f"{t}_mp_{variant}_X"], int(s[f"{t}_mp_{variant}_iters"]), A, B, C,
                     kappa=kappa_sylv(A, B))


@pytest.mark.parametrize("config,m,n", [("c0", 128, 128), ("c1", 96, 96), ("c2", 160, 96), ("c3", 96, 96),
                                         ("c0", 200, 150)])
@pytest.mark.parametrize("variant", ["orth", "inv"])
def test_against_oracle(B200, oracle, config, m, n, variant):
    from paper_2503_03456_b200 import problems as P
    pr = P.make(config, m, n, seed=0)
    ref = oracle.mp_solve(pr.A, pr.B, pr.C, variant, "binary32", pr.kind)
    p = B200.SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind)
    rep = (B200.mp_orth if variant == "orth" else B200.mp_inv)(p, cfg_for(B200, "binary32"))
    kap = kappa_sylv(pr.A, pr.B) if m * n <= 4096 else 20.0  # survey: kappa_2(M_f) <= 10 for these recipes
    check_parity(rep, ref["X"], ref["iterations"], pr.A, pr.B, pr.C, kappa=kap)
    if pr.kind == "lyapunov":
        X = rep.X.real
        assert np.linalg.norm(X - X.T) <= 1e-13 * np.linalg.norm(X)
    if pr.X_true is not None:
        assert np.linalg.norm(rep.X - pr.X_true) / np.linalg.norm(pr.X_true) < 1e-13


def test_degenerate_binary64_pair_matches_kronecker(B200, rng):
    from conftest import cmat
    cfg = B200.RefinementConfig(B200.BINARY64, B200.BINARY64)
    for solver in (B200.mp_orth, B200.mp_inv):
        A, B, C = cmat(rng, 8, 8), cmat(rng, 6, 6), cmat(rng, 8, 6)
        X_ref = np.linalg.solve(np.kron(np.eye(6), A) + np.kron(B.T, np.eye(8)), C.flatten("F")).reshape((8, 6),
                                                                                                       order="F")
        rep = solver(B200.SylvesterProblem(A, B, C), cfg)
        assert rep.converged and rep.iterations <= 2
        assert np.linalg.norm(rep.X - X_ref) <= 1e-12 * np.linalg.norm(X_ref)
        assert rep.residual <= 1e-14


def test_lyapunov_kind_and_typed_failures(B200, rng, golden_solves):
    from conftest import cmat, hermitian
    cfg = B200.RefinementConfig(B200.BINARY32, B200.BINARY64)
    A = cmat(rng, 7, 7) + 4 * np.eye(7)
    p = B200.SylvesterProblem(A, A.conj().T, hermitian(rng, 7), kind="lyapunov")
    for solver in (B200.mp_orth, B200.mp_inv):
        rep = solver(p, cfg)
        assert rep.converged and rep.residual <= 1e-14
    s = golden_solves
    ps = B200.SylvesterProblem(s["sing_A"], s["sing_B"], s["sing_C"])
    for solver, name in ((B200.mp_orth, "mp_orth"), (B200.mp_inv, "mp_inv")):
        rep = solver(ps, cfg)
        assert not rep.converged and rep.failure is not None
        assert "initial triangular solve" in rep.failure
        assert rep.failure.startswith(("singular_equation", "nan_breakdown"))
        assert np.isnan(rep.X).all()
        rep = solver(ps, cfg, y0_zero=True)
        assert not rep.converged and "refinement" in rep.failure


def test_unsupported_pair_is_rejected(B200, rng):
    from conftest import cmat
    p = B200.SylvesterProblem(cmat(rng, 4, 4), cmat(rng, 3, 3), cmat(rng, 4, 3))
    with pytest.raises(B200.UnsupportedPrecisionError):
        B200.mp_orth(p, B200.RefinementConfig(B200.TF32, B200.BINARY64))


def test_stationary_refinement_matches_oracle(B200, oracle, golden_kernels):
    k = golden_kernels
    cfg = B200.RefinementConfig(B200.BINARY64, B200.BINARY64, epsilon=1e-14, max_iter=30)
    rep = B200.solve_pert_sylv_tri_stat(k["stat_TA"], k["stat_dA"], k["stat_TB"], k["stat_dB"], k["stat_C"],
                                        np.zeros((6, 4)), cfg)
    assert rep.iterations == int(k["stat_iters"]) and rep.converged
    assert np.linalg.norm(rep.X - k["stat_X"]) <= 1e-13 * np.linalg.norm(k["stat_X"])
    # scalar fixed point (pkg/tests/test_refinement.py:80-92): contraction 0.02
    cfg = B200.RefinementConfig(B200.BINARY64, B200.BINARY64, epsilon=1e-15, max_iter=40)
    rep = B200.solve_pert_sylv_tri_stat(np.array([[2.0]]), np.array([[0.1]]), np.array([[3.0]]),
                                        np.array([[0.0]]), np.array([[10.5]]), np.array([[0.0]]), cfg)
    assert rep.converged and rep.X[0, 0].real == pytest.approx(10.5 / 5.1, rel=1e-14)
    for i in range(1, 4):
        assert rep.correction_norms[i + 1] / rep.correction_norms[i] == pytest.approx(0.02, rel=0.1)
    # divergence when the perturbation exceeds sep (test_refinement.py:94-101)
    cfg = B200.RefinementConfig(B200.BINARY64, B200.BINARY64, epsilon=1e-12, max_iter=15)
    rep = B200.solve_pert_sylv_tri_stat(np.array([[1.0]]), np.array([[0.5]]), np.array([[-0.9]]),
                                        np.array([[0.0]]), np.array([[1.0]]), np.array([[0.0]]), cfg)
    assert not rep.converged and rep.correction_norms[-1] > rep.correction_norms[0]


@pytest.mark.parametrize("variant", ["orth", "inv"])
def test_batched_matches_single_solves(B200, variant):
    """C4 path: the lane executor returns, equation by equation, exactly what the
    single-equation driver returns (same kernels, deterministic reductions)."""
    import torch
    from paper_2503_03456_b200 import problems as P
    nb, m = 6, 96
    probs = [P.make_c4(i, m) for i in range(nb)]
    A = torch.stack([torch.as_tensor(p.A) for p in probs]).cuda()
    B = torch.stack([torch.as_tensor(p.B) for p in probs]).cuda()
    C = torch.stack([torch.as_tensor(p.C) for p in probs]).cuda()
    X, reps = B200.solve_batched(A, B, C, variant=variant, lanes=4)
    assert len(reps) == nb
    for i in range(nb):
        Xi, ri = B200.solve(A[i], B[i], C[i], variant=variant)
        assert reps[i].status == 0 and reps[i].iterations == ri.iterations == 2
        assert torch.equal(X[i], Xi)
        An, Bn, Cn = probs[i].A, probs[i].B, probs[i].C
        assert backward(An, Bn, Cn, X[i].cpu().numpy()) < 1e-15


def test_batched_c4_size_against_oracle(B200, oracle):
    """Full-size C4 equations (m = n = 512) through the batched path; equation 0 vs the oracle's Alg. 3."""
    import torch
    from paper_2503_03456_b200 import problems as P
    probs = [P.make_c4(i, 512) for i in range(2)]
    A = torch.stack([torch.as_tensor(p.A) for p in probs]).cuda()
    B = torch.stack([torch.as_tensor(p.B) for p in probs]).cuda()
    C = torch.stack([torch.as_tensor(p.C) for p in probs]).cuda()
    X, reps = B200.solve_batched(A, B, C, lanes=2)
    for i, p in enumerate(probs[:1]):
        ref = oracle.mp_solve(p.A, p.B, p.C, "orth", "binary32")
        assert abs(reps[i].iterations - ref["iterations"]) <= 1
        be_ref = backward(p.A, p.B, p.C, ref["X"].real)
        assert backward(p.A, p.B, p.C, X[i].cpu().numpy()) <= 10 * max(be_ref, U64)


@pytest.mark.parametrize("config,m,n", [("c0", 300, 200), ("c3", 160, 160), ("c2", 700, 400)])
def test_factored_solve_matches_oracle(B200, oracle, config, m, n):
    """sylv_solve_factored (the 2-GPU split's second half) with Schur factors computed separately
    (split2.solve_factored): same bars against the oracle as the fused solve."""
    import torch
    from paper_2503_03456_b200 import device as D, problems as P
    from paper_2503_03456_b200.linalg import schur_tensor
    from paper_2503_03456_b200.split2 import solve_factored
    pr = P.make(config, m, n, seed=1)
    cx = pr.is_complex
    dth, dtl = (torch.complex128, torch.complex64) if cx else (torch.float64, torch.float32)
    dev = D.device()
    cv = (lambda M, dt: D.to_cm(M if cx else np.real(M), dt, dev))
    TA, UA = schur_tensor(cv(pr.A, dtl))
    TB, UB = schur_tensor(cv(pr.B, dtl))
    for variant in ("orth", "inv"):
        X, rep = solve_factored(cv(pr.A, dth), cv(pr.B, dth), cv(pr.C, dth), TA, UA, TB, UB, variant=variant)
        assert rep.status == 0
        ref = oracle.mp_solve(pr.A, pr.B, pr.C, variant, "binary32")
        Xn = D.from_cm(X)
        assert abs(rep.iterations - ref["iterations"]) <= 1
        assert backward(pr.A, pr.B, pr.C, Xn) <= 10 * max(backward(pr.A, pr.B, pr.C, ref["X"]), U64)
