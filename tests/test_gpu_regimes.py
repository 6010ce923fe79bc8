"""The reference's robustness / conditioning-regime tests, restated against the B200 path.

Problems come from problems.generate, which reproduces the reference's
``cli.generate`` byte for byte (tests/test_host.py pins it), so each test runs on
exactly the matrices the reference's own test uses.  Sources:
  criterion 3   pkg/tests/test_acceptance.py:118-137  (50 problems, residual regime)
  criterion 4   pkg/tests/test_acceptance.py:140-173  (conditioning sweep frontier)
  t=2 / t=12    pkg/tests/test_refinement.py:187-201
  orth vs inv   pkg/tests/test_refinement.py:235-241
plus a sweep at m = n = 72 (past the Kronecker cap) where every t in 0..8 is compared
with the oracle's iteration count (+-1) and failure class, real and complex.
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


def _cfg(M):
    return M.RefinementConfig(M.BINARY32, M.BINARY64)


def _gen(kind, m, n, t, seed, stream=0):
    from paper_2503_03456_b200.problems import ProblemGenerator, generate
    return generate(ProblemGenerator(kind, m, n, t, seed, stream))


def _sp(M, p):
    return M.SylvesterProblem(p.A, p.B, p.C, kind=p.kind)


def test_criterion_3_residual_regime(B200):
    cfg = _cfg(B200)
    solved = attempts = 0
    while solved < 50 and attempts < 400:
        attempts += 1
        t = float(attempts % 6)
        m = n = 6 + attempts % 7
        p = _gen("logspace-conditioned", m, n, t, 31, attempts)
        K = np.kron(np.eye(n), p.A) + np.kron(p.B.T, np.eye(m))
        if np.linalg.cond(K, np.inf) > 1e6:
            continue
        solved += 1
        for solver in (B200.mp_orth, B200.mp_inv):
            rep = solver(_sp(B200, p), cfg)
            assert rep.failure is None, (attempts, rep.failure)
            assert rep.iterations <= 10
            assert rep.residual <= 1e3 * max(m, n) * U64, (attempts, rep.residual)
    assert solved == 50


def test_criterion_4_conditioning_sweep(B200, tmp_path):
    from paper_2503_03456_b200.harness import SWEEP_COLUMNS, run_sweep_cond
    rows = run_sweep_cond(10, 10, list(range(0, 16)), 1, _cfg(B200), tmp_path / "sweep.csv", reproducible=True)
    table = [dict(zip(SWEEP_COLUMNS, r)) for r in rows]
    for row in table:
        t = row["t"]
        if t <= 7:
            assert row["r_or"] <= 1e-11 and row["r_in"] <= 1e-11, (t, row)
            assert "or:" not in row["status"] and "in:" not in row["status"], (t, row)
        if t >= 12:
            assert "or:" in row["status"] or row["r_or"] > 1e-8, (t, row)
            assert "in:" in row["status"] or row["r_in"] > 1e-8, (t, row)

    def frontier(key):
        last = -1
        for row in table:
            if row[key] is not None and np.isfinite(row[key]) and row[key] <= 1e-8:
                last = row["t"]
            else:
                break
        return last

    assert frontier("r_gmres_uh") > frontier("r_gmres_ul")
    text = (tmp_path / "sweep.csv").read_text()
    assert text.startswith("# generator = philox4x64-10\n") and "\nt,condu,res_sylv," in text


@pytest.mark.parametrize("variant", ["orth", "inv"])
def test_logspace_t2_recovers_binary64_and_t12_fails(B200, variant):
    solver = B200.mp_orth if variant == "orth" else B200.mp_inv
    rep = solver(_sp(B200, _gen("logspace-conditioned", 10, 10, 2.0, 7)), _cfg(B200))
    assert rep.converged and rep.iterations <= 4 and rep.residual <= 1e-14
    rep = solver(_sp(B200, _gen("logspace-conditioned", 10, 10, 12.0, 7)), _cfg(B200))
    assert (not rep.converged) or rep.residual > 100 * U64


def test_iteration_counts_close_between_variants(B200):
    for t in (1.0, 3.0, 5.0):
        p = _sp(B200, _gen("logspace-conditioned", 8, 8, t, 11))
        a, b = B200.mp_orth(p, _cfg(B200)), B200.mp_inv(p, _cfg(B200))
        assert abs(a.iterations - b.iterations) <= 2, (t, a.iterations, b.iterations)


def _complexify(p, seed):
    """A complex logspace problem: the same spectra 10^linspace(0, t) under complex unitary
    similarities, complex C (an extension of the reference's real generator)."""
    rng = np.random.default_rng(seed)

    def unitary(k):
        Q, R = np.linalg.qr(rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k)))
        return Q * (np.diag(R) / np.abs(np.diag(R)))[None, :]

    Qa, Qb = unitary(p.m), unitary(p.n)
    A = Qa @ p.A @ Qa.conj().T
    B = Qb @ p.B @ Qb.conj().T
    C = p.C + 1j * rng.standard_normal(p.C.shape)
    return A, B, C


@pytest.mark.parametrize("variant", ["orth", "inv"])
@pytest.mark.parametrize("cplx", [False, True])
def test_logspace_sweep_m72_against_oracle(B200, oracle, variant, cplx):
    """Iterations within +-1 of the reference algorithm for every t in 0..8, and the same
    outcome class (converged / typed failure) where the reference fails."""
    solver = B200.mp_orth if variant == "orth" else B200.mp_inv
    for t in range(0, 9):
        p = _gen("logspace-conditioned", 72, 72, float(t), 5, t)
        A, B, C = _complexify(p, 100 + t) if cplx else (p.A, p.B, p.C)
        ref = oracle.mp_solve(A, B, C, variant, "binary32")
        rep = solver(B200.SylvesterProblem(A, B, C), _cfg(B200))
        if ref["failure"] is None:
            assert rep.failure is None, (t, rep.failure)
            assert abs(rep.iterations - ref["iterations"]) <= 1, (t, rep.iterations, ref["iterations"])
            assert rep.residual <= 10 * max(ref["residual"], U64), (t, rep.residual, ref["residual"])
        else:
            assert rep.failure is not None, (t, ref["failure"])
            assert rep.failure.split(":")[0].split()[0] == ref["failure"].split()[0], (t, rep.failure, ref["failure"])
