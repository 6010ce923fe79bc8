"""Pin the CPU oracle (oracle/mpsylv_oracle.c) against the reference's own outputs.

The fixtures were produced by running the Python reference (tests/golden/make_golden.py).
binary32 paths must match BIT FOR BIT (simulated binary32 == IEEE binary32 without FMA);
binary64 paths call numpy/OpenBLAS in the reference and agree to a few ulps.
"""

import numpy as np
import pytest

FMTS = ["binary32", "binary64"]


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def tol(name, bits64=1e-14):
    return 0.0 if name == "binary32" else bits64


@pytest.mark.parametrize("name", FMTS)
def test_gemm(oracle, golden_kernels, name):
    k = golden_kernels
    f = name == "binary32"
    A, B, C = k[f"gemm_{name}_A"], k[f"gemm_{name}_B"], k[f"gemm_{name}_C"]
    assert rel(oracle.gemm(1, A, B, 0, None, f), k[f"gemm_{name}_ab"]) <= tol(name)
    assert rel(oracle.gemm(-1, A, B, 1, C, f), k[f"gemm_{name}_neg"]) <= tol(name)


@pytest.mark.parametrize("name", FMTS)
@pytest.mark.parametrize("tag", ["real", "cplx", "c0"])
def test_hessenberg_and_schur(oracle, golden_kernels, name, tag):
    k = golden_kernels
    f = name == "binary32"
    M = k[f"schur_{name}_{tag}_in"]
    H, U = oracle.hessenberg(M, f)
    assert rel(H, k[f"hess_{name}_{tag}_H"]) <= tol(name, 1e-13)
    assert rel(U, k[f"hess_{name}_{tag}_U"]) <= tol(name, 1e-13)
    U2, T2, _ = oracle.schur(M, f)
    # binary64 Schur vectors amplify last-ulp differences of the BLAS-based reference
    assert rel(T2, k[f"schur_{name}_{tag}_T"]) <= tol(name, 1e-10)
    assert rel(U2, k[f"schur_{name}_{tag}_U"]) <= tol(name, 1e-10)


@pytest.mark.parametrize("name", FMTS)
def test_mgs_qr_lu_tri(oracle, golden_kernels, name):
    k = golden_kernels
    f = name == "binary32"
    Q, R = oracle.mgs_qr(k[f"qr_{name}_in"], f)
    assert rel(Q, k[f"qr_{name}_Q"]) <= tol(name) and rel(R, k[f"qr_{name}_R"]) <= tol(name)
    W, piv = oracle.lu(k[f"lu_{name}_in"], f)
    assert rel(W, k[f"lu_{name}_lu"]) <= tol(name) and (piv == k[f"lu_{name}_piv"]).all()
    for side, tr, rhs in (("left", "no", "rhs"), ("left", "conj", "rhs"), ("right", "no", "rhsr"),
                          ("right", "conj", "rhsr")):
        X = oracle.lu_solve(W, piv, k[f"lu_{name}_{rhs}"], side, tr, f)
        assert rel(X, k[f"lu_{name}_{side}_{tr}"]) <= tol(name, 1e-13)
    TA = k[f"tri_{name}_TA"]
    Y = oracle.solve_sylv_tri(TA, k[f"tri_{name}_TB"], k[f"tri_{name}_W"], f)
    assert rel(Y, k[f"tri_{name}_Y"]) <= tol(name)
    Y2 = oracle.solve_sylv_tri(TA, TA.conj().T, k[f"tri_{name}_W2"], f)
    assert rel(Y2, k[f"tri_{name}_Ylow"]) <= tol(name)


def test_stationary_refinement(oracle, golden_kernels):
    k = golden_kernels
    r = oracle.stat(k["stat_TA"], k["stat_dA"], k["stat_TB"], k["stat_dB"], k["stat_C"], np.zeros((6, 4)),
                    1e-14, 30)
    assert r["iterations"] == int(k["stat_iters"])
    assert rel(r["X"], k["stat_X"]) <= 1e-14
    # corrections below ~1e-12 relative are rounding noise of the binary64 loop
    np.testing.assert_allclose(r["correction_norms"], k["stat_norms"], rtol=1e-8,
                               atol=1e-13 * k["stat_norms"][0])


def _solve_tags(s):
    return sorted({key.rsplit("_", 1)[0] for key in s.files if key.endswith("_kind")})


@pytest.mark.parametrize("variant", ["orth", "inv"])
def test_mixed_precision_solves(oracle, golden_solves, variant):
    s = golden_solves
    for t in _solve_tags(s):
        r = oracle.mp_solve(s[f"{t}_A"], s[f"{t}_B"], s[f"{t}_C"], variant, str(s[f"{t}_ul"]),
                            str(s[f"{t}_kind"]))
        Xr = s[f"{t}_mp_{variant}_X"]
        assert r["iterations"] == int(s[f"{t}_mp_{variant}_iters"]), t
        assert rel(r["X"], Xr) <= 1e-13, t
        ref_norms = s[f"{t}_mp_{variant}_norms"]
        # D_1 is the binary32 error of Y0: identical bits give identical norms
        if str(s[f"{t}_ul"]) == "binary32":
            assert abs(r["correction_norms"][0] / ref_norms[0] - 1) < 1e-9, t
        assert abs(r["residual"] - float(s[f"{t}_mp_{variant}_res"])) <= 1e-15, t


@pytest.mark.parametrize("variant", ["orth", "inv"])
@pytest.mark.parametrize("y0", [0, 1])
def test_typed_failures(oracle, golden_solves, variant, y0):
    s = golden_solves
    r = oracle.mp_solve(s["sing_A"], s["sing_B"], s["sing_C"], variant, "binary32", y0_zero=y0)
    ref = str(s[f"sing_mp_{variant}_{y0}_fail"])
    assert r["failure"] is not None and ref.startswith(r["failure"])
    if not y0:
        assert np.isnan(r["X"]).all()
