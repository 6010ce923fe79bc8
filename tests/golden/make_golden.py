"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

This script imports the read-only Python reference ``mpsylv`` from
``/root/reference/pkg/src`` (it only exists in the build container, never on
the GPU box) and records inputs and outputs of the hot-path functions at
sizes the reference finishes in seconds.  The committed ``.npz`` files are
what the tests read; re-run with

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Functions pinned (reference file:line):
  gemm            pkg/src/mpsylv/linalg.py:125-154
  _hessenberg     pkg/src/mpsylv/linalg.py:446-464
  schur           pkg/src/mpsylv/linalg.py:518-577
  mgs_qr          pkg/src/mpsylv/linalg.py:252-273
  lu / lu_solve   pkg/src/mpsylv/linalg.py:349-440
  solve_sylv_tri  pkg/src/mpsylv/sylvester.py:111-157
  solve_pert_sylv_tri_stat  pkg/src/mpsylv/refinement.py:95-141
  mp_orth / mp_inv          pkg/src/mpsylv/refinement.py:205-297
  residual        pkg/src/mpsylv/sylvester.py:199-209
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import mpsylv  # noqa: E402  (reference, read-only)
from mpsylv import linalg as L  # noqa: E402
from mpsylv.precision import BINARY32, BINARY64, PrecisionContext  # noqa: E402
from mpsylv.refinement import RefinementConfig, mp_inv, mp_orth, solve_pert_sylv_tri_stat  # noqa: E402
from mpsylv.sylvester import SylvesterProblem, residual, solve_sylv_tri  # noqa: E402

from paper_2503_03456_b200 import problems  # noqa: E402

C32 = PrecisionContext(BINARY32)
C64 = PrecisionContext(BINARY64)
FMT = {"binary32": C32, "binary64": C64}


def cmat(rng, m, n):
    return rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))


def kernels():
    """Component KATs: gemm, hessenberg, schur, mgs_qr, lu, lu_solve, tri-solve."""
    rng = np.random.default_rng(20240901)
    out = {}
    for name, ctx in FMT.items():
        # gemm: complex, alpha/beta variants (values representable in binary32)
        A = L._round_complex_array(cmat(rng, 7, 5), ctx.format)
        B = L._round_complex_array(cmat(rng, 5, 6), ctx.format)
        Cm = L._round_complex_array(cmat(rng, 7, 6), ctx.format)
        out[f"gemm_{name}_A"], out[f"gemm_{name}_B"], out[f"gemm_{name}_C"] = A, B, Cm
        out[f"gemm_{name}_ab"] = L.gemm(1.0, A, B, 0.0, None, ctx)
        out[f"gemm_{name}_neg"] = L.gemm(-1.0, A, B, 1.0, Cm, ctx)
        # hessenberg + schur on real and complex inputs
        for tag, M in (("real", rng.standard_normal((12, 12)) + 0j),
                       ("cplx", cmat(rng, 10, 10)),
                       ("c0", problems.make_c0(16, 16, seed=3).A + 0j)):
            Mi = L._enter(M, ctx)
            H, U = L._hessenberg(Mi, ctx)
            sf = L.schur(M, ctx)
            out[f"schur_{name}_{tag}_in"] = M
            out[f"hess_{name}_{tag}_H"] = H
            out[f"hess_{name}_{tag}_U"] = U
            out[f"schur_{name}_{tag}_T"] = sf.T
            out[f"schur_{name}_{tag}_U"] = sf.U
        # mgs_qr of a near-unitary factor and of a random matrix
        sf = L.schur(cmat(rng, 9, 9), C32)
        out[f"qr_{name}_in"] = sf.U
        f = L.mgs_qr(sf.U, ctx)
        out[f"qr_{name}_Q"], out[f"qr_{name}_R"] = f.Q, f.R
        # lu + the four lu_solve modes
        M = L._round_complex_array(cmat(rng, 8, 8), ctx.format)
        R = L._round_complex_array(cmat(rng, 8, 3), ctx.format)
        Rr = L._round_complex_array(cmat(rng, 3, 8), ctx.format)
        F = L.lu(M, ctx)
        out[f"lu_{name}_in"], out[f"lu_{name}_rhs"], out[f"lu_{name}_rhsr"] = M, R, Rr
        out[f"lu_{name}_lu"], out[f"lu_{name}_piv"] = F.lu, F.pivots
        for side, tr in (("left", "no"), ("left", "conj")):
            out[f"lu_{name}_{side}_{tr}"] = L.lu_solve(F, R, side, tr, ctx)
        for side, tr in (("right", "no"), ("right", "conj")):
            out[f"lu_{name}_{side}_{tr}"] = L.lu_solve(F, Rr, side, tr, ctx)
        # triangular Sylvester: upper/upper and upper/lower (Lyapunov adjoint)
        TA = L._round_complex_array(np.triu(cmat(rng, 9, 9)) + 3 * np.eye(9), ctx.format)
        TB = L._round_complex_array(np.triu(cmat(rng, 6, 6)) + 3 * np.eye(6), ctx.format)
        W = L._round_complex_array(cmat(rng, 9, 6), ctx.format)
        out[f"tri_{name}_TA"], out[f"tri_{name}_TB"], out[f"tri_{name}_W"] = TA, TB, W
        out[f"tri_{name}_Y"] = solve_sylv_tri(TA, TB, W, ctx)
        TL = TA.conj().T.copy()
        W2 = L._round_complex_array(cmat(rng, 9, 9), ctx.format)
        out[f"tri_{name}_W2"] = W2
        out[f"tri_{name}_Ylow"] = solve_sylv_tri(TA, TL, W2, ctx)
    # the stationary refinement loop (binary64, Alg. 1)
    TA = np.triu(cmat(rng, 6, 6)) + 3 * np.eye(6)
    TB = np.triu(cmat(rng, 4, 4)) + 3 * np.eye(4)
    dA, dB = 0.05 * cmat(rng, 6, 6), 0.05 * cmat(rng, 4, 4)
    Cm = cmat(rng, 6, 4)
    cfg = RefinementConfig(BINARY64, BINARY64, epsilon=1e-14, max_iter=30)
    rep = solve_pert_sylv_tri_stat(TA, dA, TB, dB, Cm, np.zeros((6, 4)), cfg)
    out.update(stat_TA=TA, stat_TB=TB, stat_dA=dA, stat_dB=dB, stat_C=Cm,
               stat_X=rep.X, stat_iters=rep.iterations,
               stat_norms=np.array(rep.correction_norms), stat_res=rep.residual)
    return out


SOLVES = [
    # (tag, config, m, n, seed, ul)
    ("c0_16", "c0", 16, 16, 0, "binary32"),
    ("c0_24x20", "c0", 24, 20, 1, "binary32"),
    ("c0_32", "c0", 32, 32, 0, "binary32"),
    ("c1_16", "c1", 16, 16, 0, "binary32"),
    ("c1_24", "c1", 24, 24, 2, "binary32"),
    ("c2_20x12", "c2", 20, 12, 0, "binary32"),
    ("c3_12", "c3", 12, 12, 0, "binary32"),
    ("c3_16x10", "c3", 16, 10, 1, "binary32"),
    ("c0_12_f64", "c0", 12, 12, 0, "binary64"),
    ("c1_12_f64", "c1", 12, 12, 0, "binary64"),
]


def solves():
    out = {}
    for tag, cfgname, m, n, seed, ul in SOLVES:
        pr = problems.make(cfgname, m, n, seed=seed)
        p = SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind)
        cfg = RefinementConfig(FMT[ul].format, BINARY64)
        out[f"{tag}_A"], out[f"{tag}_B"], out[f"{tag}_C"] = pr.A, pr.B, pr.C
        out[f"{tag}_kind"] = np.array(pr.kind)
        out[f"{tag}_ul"] = np.array(ul)
        for solver in (mp_orth, mp_inv):
            t0 = time.time()
            rep = solver(p, cfg)
            s = solver.__name__
            out[f"{tag}_{s}_X"] = rep.X
            out[f"{tag}_{s}_iters"] = rep.iterations
            out[f"{tag}_{s}_norms"] = np.array(rep.correction_norms)
            out[f"{tag}_{s}_res"] = rep.residual
            out[f"{tag}_{s}_conv"] = rep.converged
            out[f"{tag}_{s}_fail"] = np.array(rep.failure or "")
            print(f"{tag} {s}: k={rep.iterations} res={rep.residual:.2e} "
                  f"({time.time() - t0:.1f}s)", flush=True)
    # typed failure: singular equation at the initial solve (refinement.py:237-241)
    rng = np.random.default_rng(20240901)
    A = np.triu(cmat(rng, 3, 3))
    B = np.triu(cmat(rng, 2, 2))
    A[0, 0], B[0, 0] = 1.0, -1.0
    p = SylvesterProblem(A, B, np.ones((3, 2)))
    out["sing_A"], out["sing_B"], out["sing_C"] = p.A, p.B, p.C
    for solver in (mp_orth, mp_inv):
        for y0z in (False, True):
            rep = solver(p, RefinementConfig(BINARY32, BINARY64), y0_zero=y0z)
            key = f"sing_{solver.__name__}_{int(y0z)}"
            out[f"{key}_fail"] = np.array(rep.failure or "")
            out[f"{key}_iters"] = rep.iterations
    return out


def main():
    t0 = time.time()
    k = kernels()
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **k)
    print(f"kernels.npz: {len(k)} arrays ({time.time() - t0:.1f}s)", flush=True)
    s = solves()
    np.savez_compressed(os.path.join(HERE, "solves.npz"), **s)
    print(f"solves.npz: {len(s)} arrays ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
