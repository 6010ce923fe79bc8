"""Harness / wire-format parity: Matrix Market I/O, CSV metadata,
generators, CLI parsing -- host logic, no GPU needed.  The GPU-driven sweeps are in
tests/test_gpu_regimes.py (criterion 4) and test_gpu_harness below."""

import os

import numpy as np
import pytest

from paper_2503_03456_b200 import harness as H
from paper_2503_03456_b200.mmio import read_matrix, write_matrix


def test_matrix_market_round_trip_is_bit_exact(tmp_path, rng):
    M = rng.standard_normal((7, 5)) + 1j * rng.standard_normal((7, 5))
    M[2, 3] = np.nextafter(1.0, 2.0) + 1e-300j
    write_matrix(tmp_path / "m.mtx", M)
    R = read_matrix(tmp_path / "m.mtx")
    assert R.dtype == np.complex128 and np.array_equal(R.view(np.uint64), M.view(np.uint64))
    write_matrix(tmp_path / "d.mtx", M, hexfloat=False)
    assert np.array_equal(read_matrix(tmp_path / "d.mtx"), M)


@pytest.mark.parametrize("sym", ["symmetric", "hermitian", "skew-symmetric"])
def test_matrix_market_symmetric_coordinate_and_array(tmp_path, sym):
    coord = tmp_path / "c.mtx"
    coord.write_text(f"%%MatrixMarket matrix coordinate complex {sym}\n% comment\n3 3 3\n"
                     "1 1 2.0 0.0\n3 1 0x1.8p+0 -1.0\n2 2 -4 0\n")
    M = read_matrix(coord)
    v = complex(1.5, -1.0)
    mirror = {"symmetric": v, "hermitian": v.conjugate(), "skew-symmetric": -v}[sym]
    assert M[2, 0] == v and M[0, 2] == mirror and M[0, 0] == 2 and M[1, 1] == -4
    arr = tmp_path / "a.mtx"
    arr.write_text("%%MatrixMarket matrix array real symmetric\n2 2\n1\n2\n3\n")
    A = read_matrix(arr)
    assert np.array_equal(A, np.array([[1, 2], [2, 3]], dtype=complex))


def test_matrix_market_rejects_bad_headers(tmp_path):
    bad = tmp_path / "b.mtx"
    bad.write_text("%%MatrixMarket matrix array pattern general\n1 1\n1\n")
    with pytest.raises(ValueError):
        read_matrix(bad)
    bad.write_text("not a header\n")
    with pytest.raises(ValueError):
        read_matrix(bad)


def test_csv_metadata_and_reproducible_flag(tmp_path):
    from paper_2503_03456_b200 import BINARY32, BINARY64, RefinementConfig
    md = H._metadata(RefinementConfig(BINARY32, BINARY64), 20, 7, {"m": 3})
    H.write_csv(tmp_path / "r.csv", md, ["a", "b"], [[1.5, None], [float("nan"), "ok"]], reproducible=True)
    text = (tmp_path / "r.csv").read_text()
    assert text == ("# generator = philox4x64-10\n# seed = 7\n# ul = binary32\n# uh = binary64\n"
                    "# max_iter = 20\n# epsilon = auto\n# gmres_restart = 20\n# m = 3\na,b\n1.5,\nnan,ok\n")
    H.write_csv(tmp_path / "s.csv", md, ["a"], [], reproducible=False)
    assert (tmp_path / "s.csv").read_text().startswith("# written = ")


def test_cli_parser_and_helpers():
    ap = H.build_parser()
    a = ap.parse_args(["sweep-cond", "--m", "12", "--t-range", "2:5", "--out", "x.csv", "--reproducible"])
    assert a.command == "sweep-cond" and H.t_range(a.t_range) == [2, 3, 4, 5] and a.ul.name == "binary32"
    a = ap.parse_args(["solve", "--matrix-market", "A", "B", "C", "--out", "o.csv", "--solvers", "or,bs"])
    assert a.matrix_market == ["A", "B", "C"] and a.solvers == "or,bs"
    assert H.failure_slug(None) == "ok"
    assert H.failure_slug("singular_equation at initial triangular solve: x") == "singular_equation"
    assert H.failure_slug("nan_breakdown: iterate diverged") == "nan_breakdown"


def test_condu_uses_the_kronecker_operator_under_the_cap():
    from paper_2503_03456_b200 import BINARY64
    from paper_2503_03456_b200.problems import ProblemGenerator, generate
    p = generate(ProblemGenerator("logspace-conditioned", 6, 5, 2.0, 3))
    M = np.kron(np.eye(5), p.A) + np.kron(p.B.T, np.eye(6))
    assert H.condu(p, BINARY64) == pytest.approx(np.linalg.cond(M) * 2.0 ** -53, rel=1e-10)
    big = generate(ProblemGenerator("random-dense", 70, 70, 0.0, 1))
    assert H.condu(big, BINARY64) is None


@pytest.mark.gpu
def test_gpu_harness_solve_from_matrix_market(tmp_path):
    """`solve --matrix-market A B C` through the CLI entry point, every solver."""
    from paper_2503_03456_b200.problems import ProblemGenerator, generate
    p = generate(ProblemGenerator("logspace-conditioned", 12, 9, 2.0, 4))
    for name, M in (("A", p.A), ("B", p.B), ("C", p.C)):
        write_matrix(tmp_path / f"{name}.mtx", M)
    out = tmp_path / "solve.csv"
    rc = H.main(["solve", "--matrix-market", str(tmp_path / "A.mtx"), str(tmp_path / "B.mtx"),
                 str(tmp_path / "C.mtx"), "--out", str(out), "--reproducible"])
    assert rc == 0
    lines = [ln for ln in out.read_text().splitlines() if not ln.startswith("#")]
    assert lines[0] == "solver,residual,iterations,converged,status"
    rows = {r.split(",")[0]: r.split(",") for r in lines[1:]}
    assert set(rows) == set(H.ALL_SOLVERS)
    for name, r in rows.items():
        assert r[4] == "ok", r
        assert float(r[1]) <= 1e-13, r
