"""CPU-only checks: the C ABI library loads and exports every symbol the header
declares, the host-side mirror of the reference API validates like the
reference, the generators are deterministic, the cost model matches."""

import ctypes as ct
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mpsylv_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|unsigned long long)\s+(sylv_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2503_03456_b200 import _native
    from paper_2503_03456_b200.build import build
    build(verbose=False)
    lib = ct.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS)


def test_struct_layouts_match_header():
    from paper_2503_03456_b200 import _native
    # sylv_params: 9 ints + a double (aligned) ; sylv_report contains the norms array
    assert ct.sizeof(_native.Params) == 48
    assert ct.sizeof(_native.Report) > 8 * _native.MAX_NORMS


def test_status_strings_without_gpu():
    from paper_2503_03456_b200 import _native
    L = _native.lib()
    assert L.sylv_version() == 1
    assert L.sylv_status_string(1) == b"singular_equation"
    assert L.sylv_status_string(-3) == b"workspace_too_small"


def test_workspace_queries_without_gpu():
    from paper_2503_03456_b200 import _native
    L = _native.lib()
    p = _native.Params(m=4096, n=4096, kind=0, complex_data=0, variant=0, low_bits=32, correction_bits=64,
                       max_iter=20, y0_zero=0, epsilon=4.096e-9)
    sz = ct.c_size_t()
    assert L.sylv_workspace_size(ct.byref(p), ct.byref(sz)) == 0
    assert 1e9 < sz.value < 8e9
    p.low_bits = 16
    assert L.sylv_workspace_size(ct.byref(p), ct.byref(sz)) == _native.EUNSUPPORTED


def test_config_and_precision_pairs():
    from paper_2503_03456_b200 import (BFLOAT16, BINARY32, BINARY64, TF32, RefinementConfig,
                                       UnsupportedPrecisionError)
    from paper_2503_03456_b200.refinement import _precision_pair
    assert RefinementConfig(BINARY64, BINARY64).resolve_epsilon(7, 12) == 1e-12 * 12
    assert RefinementConfig(TF32, BINARY32).resolve_epsilon(5, 5) == 1e4 * BINARY32.unit_roundoff * 5
    with pytest.raises(ValueError):
        RefinementConfig(BINARY64, BINARY32)
    assert RefinementConfig(BINARY32, BINARY64).max_iter == 20
    assert _precision_pair(RefinementConfig(BINARY32, BINARY64)) == 32
    assert _precision_pair(RefinementConfig(BINARY64, BINARY64)) == 64
    for lo in (TF32, BFLOAT16):
        with pytest.raises(UnsupportedPrecisionError):
            _precision_pair(RefinementConfig(lo, BINARY64))


def test_sylvester_problem_validation(rng):
    from paper_2503_03456_b200 import DimensionError, SylvesterProblem
    A = rng.standard_normal((3, 3))
    with pytest.raises(ValueError):
        SylvesterProblem(A, A, np.ones((3, 3)), kind="lyapunov")
    with pytest.raises(DimensionError):
        SylvesterProblem(A, np.eye(2), np.ones((3, 3)))
    p = SylvesterProblem(A, A.T, np.ones((3, 3)), kind="lyapunov")
    assert p.m == 3 and p.n == 3 and p.A.dtype == np.complex128


def test_cost_model_matches_reference_table():
    from paper_2503_03456_b200.costmodel import flops
    a, b = 2 * 128 ** 3, 128 * 128 * 256
    f = flops("mp_orth_sylv", 128, 128, 2)
    assert f.low_flops == 25 * a + b and f.high_flops == 6 * a + 10 * b
    assert flops("mp_orth_lyap", 10, 10, 1).high_flops == 20 * 1000


def test_generators_deterministic_and_shaped():
    from paper_2503_03456_b200 import problems as P
    a, b = P.make("c0", 16, seed=0), P.make("c0", 16, seed=0)
    assert (a.A == b.A).all() and (a.C == b.C).all()
    c1 = P.make("c1", 12)
    assert np.allclose(c1.B, c1.A.T) and np.allclose(c1.C, c1.C.T)
    c2 = P.make("c2", 12, 8)
    assert np.linalg.norm(c2.A @ c2.X_true + c2.X_true @ c2.B - c2.C) < 1e-12 * np.linalg.norm(c2.C)
    c3 = P.make("c3", 8)
    assert c3.is_complex and not c2.is_complex
    assert (P.make_c4(3, 16).A == P.make_c0(16, 16, 3).A).all()


def test_golden_fixture_inputs_follow_generators(golden_solves):
    from paper_2503_03456_b200 import problems as P
    s = golden_solves
    p = P.make("c0", 24, 20, seed=1)
    assert np.array_equal(s["c0_24x20_A"], p.A) and np.array_equal(s["c0_24x20_C"], p.C)


def test_bartels_stewart_variant_params_without_gpu():
    """SYLV_VARIANT_BS: binary64 only (EUNSUPPORTED for low_bits 32); its workspace is the
    mp_orth one minus the B-side scratch the orth variant runs beside Schur(A)."""
    from paper_2503_03456_b200 import _native
    L = _native.lib()

    def size(variant, low_bits, kind=_native.KIND_GENERAL):
        p = _native.Params(m=300, n=200, kind=kind, complex_data=0, variant=variant, low_bits=low_bits,
                           correction_bits=64, max_iter=20, y0_zero=0, epsilon=0.0)
        sz = ct.c_size_t()
        return L.sylv_workspace_size(ct.byref(p), ct.byref(sz)), sz.value

    rc, bs = size(_native.VARIANT_BS, 64)
    assert rc == 0 and bs > 0
    assert size(_native.VARIANT_BS, 32)[0] == _native.EUNSUPPORTED
    rc, orth64 = size(_native.VARIANT_ORTH, 64)
    assert rc == 0 and orth64 > bs  # orth(B) + S_B scratch (2 n^2 doubles) beside the A side
    assert orth64 - bs >= 2 * 200 * 200 * 8


def test_kernel_timer_abi_without_gpu():
    from paper_2503_03456_b200 import _native
    L = _native.lib()
    n = 8
    c, ms, fl = (ct.c_longlong * n)(), (ct.c_double * n)(), (ct.c_double * n)()
    assert L.sylv_ktimer(1, n, c, ms, fl) == 0
    assert L.sylv_ktimer(2, n, c, ms, fl) == 0 and sum(c) == 0
    assert L.sylv_ktimer(0, n, c, ms, fl) == 0
    assert L.sylv_ktimer(7, n, c, ms, fl) == _native.EINVAL


def test_triangular_form_follows_reference_test():
    """sylvester.py:100-108: strictly triangular first; quasi forms only with isolated 2x2 blocks."""
    from paper_2503_03456_b200.errors import DimensionError
    from paper_2503_03456_b200.sylvester import _triangular_form
    up = np.triu(np.ones((5, 5)))
    assert _triangular_form(up, True) == "upper"
    lo_bidiag = np.diag(np.ones(5)) + np.diag(np.ones(4), -1)
    assert _triangular_form(lo_bidiag, True) == "lower"       # not mistaken for quasi-upper
    quasi = up.copy()
    quasi[1, 0] = quasi[4, 3] = 0.5
    assert _triangular_form(quasi, True) == "upper"
    assert _triangular_form(quasi.T, True) == "lower"
    hess = up + np.diag(np.ones(4), -1)                        # consecutive subdiagonals
    with pytest.raises(DimensionError):
        _triangular_form(hess, True)
    with pytest.raises(DimensionError):
        _triangular_form(quasi, False)
    with pytest.raises(DimensionError):
        _triangular_form(np.ones((3, 3)), True)


def test_batched_workspace_uses_effective_lanes():
    """The workspace is sized for min(lanes, batch) lanes, not the 64-lane default (a 2-equation
    batch at m=n=4096 must not ask for 64 lanes of workspace)."""
    import ctypes as ct
    from paper_2503_03456_b200 import _native
    from paper_2503_03456_b200.batch import effective_lanes, _params
    assert effective_lanes(0, 2) == 2 and effective_lanes(0, 500) == 64 and effective_lanes(8, 3) == 3
    L = _native.lib()
    p = _params(4096, 4096, False, "general", "orth", 32, 64, 1e-9, 20, False)
    one, two = ct.c_size_t(), ct.c_size_t()
    assert L.sylv_workspace_size(ct.byref(p), ct.byref(one)) == 0
    assert L.sylv_batched_workspace_size(ct.byref(p), effective_lanes(0, 2), ct.byref(two)) == 0
    assert two.value <= 2 * (one.value + 256)


def test_generators_reproduce_reference_bytes():
    """problems.generate == the reference's cli.generate, byte for byte (fixture digests made by
    running the reference: tests/golden/make_golden_generators.py)."""
    import hashlib
    import json
    from paper_2503_03456_b200.problems import ProblemGenerator, generate
    with open(os.path.join(os.path.dirname(__file__), "golden", "generators.json")) as f:
        fixtures = json.load(f)

    def digest(M):
        return hashlib.sha256(np.ascontiguousarray(np.asarray(M, dtype=np.complex128)).tobytes()).hexdigest()

    for fx in fixtures:
        p = generate(ProblemGenerator(*fx["spec"]))
        assert (digest(p.A), digest(p.B), digest(p.C)) == (fx["A"], fx["B"], fx["C"]), fx["spec"]
        assert p.kind == fx["kind"]
