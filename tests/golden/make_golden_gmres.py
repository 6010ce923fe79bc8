"""Golden fixtures for Schur-preconditioned GMRES-IR, produced by the REFERENCE.

Runs ``mpsylv.gmresir.gmres_ir_sylv`` (pkg/src/mpsylv/gmresir.py:208-278) from the read-only
reference at /root/reference/pkg/src (build container only) on seeded config recipes at
small sizes, for both GMRES precisions u_g in {binary64, binary32} with the refinement pair
(binary32, binary64), plus a problem whose preconditioner is singular (failure string).
Re-run with

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_gmres.py
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

from mpsylv.gmresir import GmresConfig, gmres_ir_sylv  # noqa: E402  (reference, read-only)
from mpsylv.precision import BINARY32, BINARY64  # noqa: E402
from mpsylv.refinement import RefinementConfig  # noqa: E402
from mpsylv.sylvester import SylvesterProblem  # noqa: E402

from paper_2503_03456_b200 import problems  # noqa: E402

CASES = [  # tag, recipe, m, n, seed, u_g
    ("c0_g64", "c0", 12, 10, 0, "binary64"),
    ("c0_g32", "c0", 12, 10, 0, "binary32"),
    ("c1_g64", "c1", 10, 10, 1, "binary64"),
    ("c3_g64", "c3", 8, 6, 3, "binary64"),
    ("c2_g32", "c2", 10, 8, 2, "binary32"),
]
FMT = {"binary32": BINARY32, "binary64": BINARY64}


def main():
    out = {}
    rcfg = RefinementConfig(BINARY32, BINARY64)
    for tag, cfg, m, n, seed, ug in CASES:
        pr = problems.make(cfg, m, n, seed=seed)
        p = SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind)
        t0 = time.time()
        rep = gmres_ir_sylv(p, GmresConfig(FMT[ug]), rcfg)
        out[f"{tag}_A"], out[f"{tag}_B"], out[f"{tag}_C"] = pr.A, pr.B, pr.C
        out[f"{tag}_kind"] = np.array(pr.kind)
        out[f"{tag}_ug"] = np.array(ug)
        out[f"{tag}_X"] = rep.X
        out[f"{tag}_outer"] = rep.outer_iterations
        out[f"{tag}_inner"] = np.array(rep.inner_iterations)
        out[f"{tag}_hist"] = np.array(rep.residual_history)
        out[f"{tag}_conv"] = rep.converged
        out[f"{tag}_fail"] = np.array(rep.failure or "")
        print(f"{tag}: outer={rep.outer_iterations} inner={rep.inner_iterations} "
              f"res={rep.residual_history[-1]:.2e} ({time.time() - t0:.1f}s)", flush=True)
    # singular preconditioner: eig(A) = {1, 2}, eig(B) = {-1}
    A = np.array([[1.0, 0.5], [0.0, 2.0]])
    B = np.array([[-1.0]])
    rep = gmres_ir_sylv(SylvesterProblem(A, B, np.ones((2, 1))), GmresConfig(BINARY64), rcfg)
    out["sing_A"], out["sing_B"] = A, B
    out["sing_fail"] = np.array(rep.failure or "")
    out["sing_outer"] = rep.outer_iterations
    print("singular:", rep.failure)
    np.savez_compressed(os.path.join(HERE, "gmres.npz"), **out)


if __name__ == "__main__":
    main()
