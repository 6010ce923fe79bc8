"""Component parity of the sm_100a kernels (GPU).

gemm vs an fp64/complex128 numpy product; trsyl vs the oracle's
solve_sylv_tri (complex triangular) and vs the defining equation (real
quasi-triangular, 2x2 blocks straddling tile edges, Lyapunov lower T_B);
schur vs the reference's invariants (pkg/tests/test_linalg.py:216-243:
reconstruction and unitarity within 100 m u, strict lower part zero,
spectrum); Cholesky-QR vs mgs_qr's contract.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from conftest import cmat, rand_upper  # noqa: E402


@pytest.fixture(scope="module")
def B200():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2503_03456_b200 as M
    from paper_2503_03456_b200 import _native
    _native.lib()
    return M


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("shape", [(67, 45, 33), (128, 128, 128), (300, 200, 150), (1, 7, 1)])
@pytest.mark.parametrize("cx", [False, True])
def test_gemm_matches_fp64_product(B200, rng, shape, cx):
    from paper_2503_03456_b200 import BINARY32, BINARY64, PrecisionContext
    m, n, k = shape
    A = cmat(rng, m, k) if cx else rng.standard_normal((m, k))
    B = cmat(rng, k, n) if cx else rng.standard_normal((k, n))
    C = cmat(rng, m, n) if cx else rng.standard_normal((m, n))
    ref = -1.0 * (A @ B) + 0.5 * C
    got = B200.gemm(-1.0, A, B, 0.5, C, PrecisionContext(BINARY64))
    assert rel(got, ref) < 1e-14
    got32 = B200.gemm(-1.0, A, B, 0.5, C, PrecisionContext(BINARY32))
    assert rel(got32, ref) < 1e-5


def test_gemm_ops_tn_nt(B200, rng):
    import torch
    from paper_2503_03456_b200 import _native
    import ctypes as ct
    for dt, npdt, code in ((torch.float64, np.float64, 1), (torch.complex128, np.complex128, 3),
                           (torch.float32, np.float32, 0), (torch.complex64, np.complex64, 2)):
        m, n, k = 70, 53, 41
        A = (cmat(rng, k, m) if code >= 2 else rng.standard_normal((k, m))).astype(npdt)
        Bm = (cmat(rng, n, k) if code >= 2 else rng.standard_normal((n, k))).astype(npdt)
        tA = torch.as_tensor(A.T.copy()).cuda()   # col-major A (k x m)
        tB = torch.as_tensor(Bm.T.copy()).cuda()  # col-major B (n x k)
        tC = torch.zeros((n, m), dtype=dt, device="cuda")
        one, zero = np.ones(1, npdt), np.zeros(1, npdt)
        for opa, opb, ref in ((b"C", b"C", A.conj().T @ Bm.conj().T), (b"T", b"T", A.T @ Bm.T)):
            rc = _native.lib().sylv_gemm(code, opa, opb, m, n, k, one.ctypes.data, tA.data_ptr(), k,
                                         tB.data_ptr(), n, zero.ctypes.data, tC.data_ptr(), m,
                                         torch.cuda.current_stream().cuda_stream)
            assert rc == 0
            got = tC.t().cpu().numpy()
            assert rel(got, ref) < (1e-5 if code in (0, 2) else 1e-13)


def test_gemm_complex128_dmma_all_ops(B200, rng):
    """complex128 GEMMs run on the DMMA tensor pipe (gemm_zdmma_kernel): every op pair, complex
    alpha / beta, ragged tile edges, against the numpy complex128 product."""
    import torch
    from paper_2503_03456_b200 import _native
    m, n, k = 131, 70, 75
    alpha = np.array([0.75 - 0.5j], np.complex128)
    beta = np.array([-0.25 + 1.5j], np.complex128)
    op = {b"N": lambda X: X, b"T": lambda X: X.T, b"C": lambda X: X.conj().T}
    for opa in (b"N", b"T", b"C"):
        for opb in (b"N", b"T", b"C"):
            A = cmat(rng, m, k) if opa == b"N" else cmat(rng, k, m)
            Bm = cmat(rng, k, n) if opb == b"N" else cmat(rng, n, k)
            C0 = cmat(rng, m, n)
            tA = torch.as_tensor(A.T.copy()).cuda()
            tB = torch.as_tensor(Bm.T.copy()).cuda()
            tC = torch.as_tensor(C0.T.copy()).cuda()
            rc = _native.lib().sylv_gemm(3, opa, opb, m, n, k, alpha.ctypes.data, tA.data_ptr(), A.shape[0],
                                         tB.data_ptr(), Bm.shape[0], beta.ctypes.data, tC.data_ptr(), m,
                                         torch.cuda.current_stream().cuda_stream)
            assert rc == 0
            ref = alpha[0] * (op[opa](A) @ op[opb](Bm)) + beta[0] * C0
            assert rel(tC.t().cpu().numpy(), ref) < 1e-14, (opa, opb)


@pytest.mark.parametrize("name", ["binary32", "binary64"])
def test_trsyl_matches_oracle_complex(B200, oracle, golden_kernels, name):
    from paper_2503_03456_b200 import BINARY32, BINARY64, PrecisionContext
    k = golden_kernels
    ctx = PrecisionContext(BINARY32 if name == "binary32" else BINARY64)
    TA, TB, W = k[f"tri_{name}_TA"], k[f"tri_{name}_TB"], k[f"tri_{name}_W"]
    tol = 1e-5 if name == "binary32" else 1e-13
    assert rel(B200.solve_sylv_tri(TA, TB, W, ctx), k[f"tri_{name}_Y"]) < tol
    Y2 = B200.solve_sylv_tri(TA, TA.conj().T, k[f"tri_{name}_W2"], ctx)
    assert rel(Y2, k[f"tri_{name}_Ylow"]) < tol


def quasi_upper(rng, n, frac=0.3):
    """Real upper quasi-triangular matrix with 2x2 blocks carrying complex pairs.

    Strictly-upper entries are N(0, 1/n) like the Schur factors of the configs, so the
    triangular recurrence stays well conditioned at any n."""
    T = np.triu(rng.standard_normal((n, n)), 1) / np.sqrt(n) + 3 * np.eye(n)
    i = 0
    while i < n - 1:
        if rng.random() < frac:
            T[i + 1, i] = -abs(rng.standard_normal()) - 0.5
            T[i, i + 1] = abs(rng.standard_normal()) + 0.5
            T[i + 1, i + 1] = T[i, i]
            i += 2
        else:
            i += 1
    return T


@pytest.mark.parametrize("m,n", [(9, 6), (64, 64), (65, 66), (130, 129), (200, 70)])
def test_trsyl_real_quasi_triangular(B200, rng, m, n):
    TA = quasi_upper(rng, m)
    TB = quasi_upper(rng, n)
    if m >= 65:  # force a 2x2 block across the first tile edge
        TA[64, 63] = -1.0; TA[63, 64] = 1.0; TA[64, 64] = TA[63, 63]
        if 65 < m: TA[65, 64] = 0.0
        TA[63, 62] = 0.0
    W = rng.standard_normal((m, n))
    Y = B200.solve_sylv_tri(TA, TB, W).real
    scale = (np.linalg.norm(TA) + np.linalg.norm(TB)) * np.linalg.norm(Y)
    assert np.linalg.norm(TA @ Y + Y @ TB - W) < 1e-14 * scale
    Y32 = B200.solve_sylv_tri(TA, TB, W, M32()).real
    assert np.linalg.norm(TA @ Y32 + Y32 @ TB - W) < 1e-5 * scale
    # Lyapunov orientation: lower T_B = T_A^T (descending columns)
    W2 = rng.standard_normal((m, m))
    Y2 = B200.solve_sylv_tri(TA, TA.T, W2).real
    scale = 2 * np.linalg.norm(TA) * np.linalg.norm(Y2)
    assert np.linalg.norm(TA @ Y2 + Y2 @ TA.T - W2) < 1e-14 * scale


def M32():
    from paper_2503_03456_b200 import BINARY32, PrecisionContext
    return PrecisionContext(BINARY32)


@pytest.mark.parametrize("m,n", [(40, 40), (33, 20), (65, 65), (150, 130), (300, 257)])
def test_trsyl_complex_upper_tiles(B200, rng, m, n):
    TA = np.triu(cmat(rng, m, m), 1) / np.sqrt(m) + (3 + 1j) * np.eye(m)
    TB = np.triu(cmat(rng, n, n), 1) / np.sqrt(n) + (2 - 0.5j) * np.eye(n)
    W = cmat(rng, m, n)
    for ctx, tol in ((None, 1e-14), (M32(), 1e-5)):
        Y = B200.solve_sylv_tri(TA, TB, W, ctx)
        scale = (np.linalg.norm(TA) + np.linalg.norm(TB)) * np.linalg.norm(Y)
        assert np.linalg.norm(TA @ Y + Y @ TB - W) < tol * scale


def test_trsyl_singular_pair_is_typed(B200):
    from paper_2503_03456_b200 import SingularEquationError
    with pytest.raises(SingularEquationError) as exc:
        B200.solve_sylv_tri(np.array([[1.0]]), np.array([[-1.0]]), np.array([[1.0]]))
    assert (exc.value.row, exc.value.col) == (0, 0)
    Y = B200.solve_sylv_tri(np.array([[2.0]]), np.array([[3.0]]), np.array([[10.0]]))
    assert Y[0, 0] == 2.0
    Y = B200.solve_sylv_tri(np.array([[1.0, 1.0], [0.0, 2.0]]), np.array([[3.0]]), np.array([[5.0], [6.0]]))
    assert np.allclose(Y.ravel(), [0.95, 1.2])


def test_trsyl_lower_bidiagonal_real_tb(B200, rng):
    """A real lower-bidiagonal T_B is the reference's 'lower' form (descending columns), not a
    quasi-triangular one; an upper-Hessenberg T_A is rejected like the reference does."""
    m, n = 7, 5
    TA = np.triu(rng.standard_normal((m, m))) + 4 * np.eye(m)
    TB = np.diag(rng.standard_normal(n) + 3) + np.diag(rng.standard_normal(n - 1), -1)
    C = rng.standard_normal((m, n))
    Y = B200.solve_sylv_tri(TA, TB, C)
    M = np.kron(np.eye(n), TA) + np.kron(TB.T, np.eye(m))
    Yref = np.linalg.solve(M, C.flatten("F")).reshape((m, n), order="F")
    assert np.abs(Y - Yref).max() <= 1e-12 * np.abs(Yref).max()
    from paper_2503_03456_b200.errors import DimensionError
    with pytest.raises(DimensionError):
        B200.solve_sylv_tri(TA + np.diag(np.ones(m - 1), -1), TB, C)


def _check_schur(A, sf, u, quasi):
    m = A.shape[0]
    T, U = sf.T, sf.U
    nA = np.linalg.norm(A)
    assert np.linalg.norm(U @ T @ U.conj().T - A) <= 100 * m * u * nA
    assert np.linalg.norm(U.conj().T @ U - np.eye(m)) <= 100 * m * u
    if quasi:
        assert (np.tril(T, -2) == 0).all()
        sub = np.diag(T, -1)
        assert not np.any((sub[:-1] != 0) & (sub[1:] != 0)), "two consecutive nonzero subdiagonals"
    else:
        assert (np.tril(T, -1) == 0).all()
    ev = np.linalg.eigvals(A)
    mine = np.linalg.eigvals(T) if quasi else np.diag(T)
    # spectra agree (matching by nearest neighbour)
    d = np.abs(mine[:, None] - ev[None, :]).min(axis=1).max()
    assert d <= 1e3 * m * u * max(1.0, np.abs(ev).max())


@pytest.mark.parametrize("m", [1, 2, 6, 17, 50, 128, 129, 200, 300, 520, 1100])
def test_schur_real_fp32(B200, rng, m):
    from paper_2503_03456_b200 import BINARY32, PrecisionContext
    A = rng.standard_normal((m, m))
    sf = B200.schur(A, PrecisionContext(BINARY32), real_form=True)
    _check_schur(A, sf, 2.0 ** -24, quasi=True)


@pytest.mark.parametrize("m", [6, 50, 96, 97, 260, 700])
def test_schur_complex_fp32(B200, rng, m):
    from paper_2503_03456_b200 import BINARY32, PrecisionContext
    A = cmat(rng, m, m)
    sf = B200.schur(A, PrecisionContext(BINARY32))
    _check_schur(A, sf, 2.0 ** -24, quasi=False)


@pytest.mark.parametrize("m", [12, 150, 400])
def test_schur_binary64(B200, rng, m):
    """Real binary64 (one-CTA and multishift paths) and complex binary64 (past its 64 one-CTA
    limit at 100: multishift with async endgame blocks)."""
    from paper_2503_03456_b200 import BINARY64, PrecisionContext
    A = rng.standard_normal((m, m))
    _check_schur(A, B200.schur(A, PrecisionContext(BINARY64), real_form=True), 2.0 ** -53, quasi=True)
    for mc in (40, 100):
        Ac = cmat(rng, mc, mc)
        _check_schur(Ac, B200.schur(Ac, PrecisionContext(BINARY64)), 2.0 ** -53, quasi=False)


def test_schur_reference_kats(B200, rng):
    from paper_2503_03456_b200 import BINARY64, PrecisionContext
    ctx = PrecisionContext(BINARY64)
    T0 = np.triu(cmat(rng, 5, 5))
    sf = B200.schur(T0, ctx)
    assert np.abs(np.sort_complex(np.diag(sf.T)) - np.sort_complex(np.diag(T0))).max() < 1e-13
    sf = B200.schur(np.array([[0.0, 1.0], [-1.0, 0.0]]), ctx, real_form=False)
    got = np.sort_complex(np.diag(sf.T))
    assert np.abs(got - np.array([-1j, 1j])).max() < 1e-14
    # the reference's default contract (pkg/tests/test_linalg.py): complex triangular T with an
    # exactly zero strictly-lower part, also for real input
    sf = B200.schur(np.array([[0.0, 1.0], [-1.0, 0.0]]), ctx)
    assert np.abs(np.sort_complex(np.diag(sf.T)) - np.array([-1j, 1j])).max() < 1e-14
    Ar = rng.standard_normal((17, 17))
    sf = B200.schur(Ar, ctx)
    assert (np.tril(sf.T, -1) == 0).all()
    A = np.eye(3, k=-1) + 0j  # companion of z^3 = 1: needs exceptional shifts
    A[0, 2] = 1.0
    sf = B200.schur(A, ctx, real_form=False)
    got = np.sort_complex(np.diag(sf.T))
    assert np.abs(got - np.sort_complex(np.exp(2j * np.pi * np.arange(3) / 3))).max() < 1e-10


@pytest.mark.parametrize("m", [9, 64, 100, 300])
def test_orth_cholesky_qr(B200, rng, m):
    from paper_2503_03456_b200 import BINARY32, PrecisionContext
    A = rng.standard_normal((m, m))
    U = B200.schur(A, PrecisionContext(BINARY32), real_form=True).U.real
    f = B200.mgs_qr(U)
    Q, R = f.Q.real, f.R.real
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) < 1e-13 * m
    assert np.linalg.norm(Q @ R - U) < 1e-13 * m
    assert (np.diag(R) > 0).all() and (np.tril(R, -1) == 0).all()
    Uc = B200.schur(cmat(rng, m, m), PrecisionContext(BINARY32)).U
    fc = B200.mgs_qr(Uc)
    assert np.linalg.norm(fc.Q.conj().T @ fc.Q - np.eye(m)) < 1e-13 * m
    assert np.linalg.norm(fc.Q @ fc.R - Uc) < 1e-13 * m
    assert (np.diag(fc.R).real > 0).all() and np.abs(np.diag(fc.R).imag).max() < 1e-15



def test_hermitian_eig_reference_kats(B200, rng):
    """pkg/tests/test_linalg.py:246-270: identity, [[2,1],[1,2]] -> {1, 3}, random Hermitian
    reconstruction and unitarity, non-Hermitian input rejected."""
    U, d = B200.hermitian_eig(np.eye(3))
    assert np.allclose(np.sort(d), 1.0) and np.allclose(U.conj().T @ U, np.eye(3))
    U, d = B200.hermitian_eig(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(np.sort(d), [1.0, 3.0], atol=1e-14)
    for n in (9, 40, 150):
        H = cmat(rng, n, n)
        H = (H + H.conj().T) / 2
        U, d = B200.hermitian_eig(H)
        assert np.linalg.norm(U @ np.diag(d) @ U.conj().T - H) <= 100 * n * 2.0 ** -53 * np.linalg.norm(H)
        assert np.linalg.norm(U.conj().T @ U - np.eye(n)) <= 100 * n * 2.0 ** -53
        assert np.allclose(np.sort(d), np.linalg.eigvalsh(H), atol=1e-12 * np.abs(d).max())
    from paper_2503_03456_b200.errors import NotHermitianError
    with pytest.raises(NotHermitianError):
        B200.hermitian_eig(cmat(rng, 4, 4))


@pytest.mark.parametrize("m,n,cplx", [(7, 5, True), (60, 45, False), (300, 200, False)])
def test_solve_hermitian_matches_kronecker(B200, rng, m, n, cplx):
    """solve_hermitian (sylvester.py:181-196) against the explicit Kronecker solve
    (pkg/tests/test_sylvester.py:150-165 and acceptance criterion 2, test_acceptance.py:85-115)."""
    def herm(k, shift):
        G = cmat(rng, k, k) if cplx else rng.standard_normal((k, k))
        return (G + G.conj().T) / 2 + shift * np.eye(k)
    A, B = herm(m, 3.0 + np.sqrt(m)), herm(n, 1.0 + np.sqrt(n))
    C = cmat(rng, m, n) if cplx else rng.standard_normal((m, n))
    p = B200.SylvesterProblem(A, B, C, kind="hermitian")
    X = B200.solve_hermitian(p)
    if m * n <= 4096:
        Xk = np.linalg.solve(np.kron(np.eye(n), A) + np.kron(B.T, np.eye(m)), C.flatten("F")).reshape((m, n), order="F")
        assert np.linalg.norm(X - Xk) <= 1e-11 * np.linalg.norm(Xk)
    assert B200.residual(p, X) <= 1e-14
    with pytest.raises(ValueError):
        B200.solve_hermitian(B200.SylvesterProblem(A, B, C))
    # exactly singular: spec(A) meets spec(-B)
    with pytest.raises(B200.SingularEquationError):
        B200.solve_hermitian(B200.SylvesterProblem(np.diag([1.0, 2.0]), np.diag([-2.0]), np.ones((2, 1)),
                                                   kind="hermitian"))


@pytest.mark.gpu
def test_schur_run_to_run_identical():
    """The large Schur runs detached blocks on helper threads and far applications on side
    streams; every entry still receives its operations in one fixed order, so two runs of the
    same matrix agree bit for bit (a race between the streams would show up here)."""
    import torch
    from paper_2503_03456_b200.linalg import schur_tensor
    torch.manual_seed(5)
    m = 1500
    A = (torch.randn(m, m, device="cuda", dtype=torch.float64) / m ** 0.5 + 2 * torch.eye(m, device="cuda",
                                                                                       dtype=torch.float64)).float()
    T1, U1 = schur_tensor(A.clone(), [])
    T2, U2 = schur_tensor(A.clone(), [])
    torch.cuda.synchronize()
    assert torch.equal(T1, T2) and torch.equal(U1, U2)
