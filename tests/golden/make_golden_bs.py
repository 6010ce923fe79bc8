"""Golden fixtures for the fp64 Bartels-Stewart comparator, produced by the REFERENCE.

Runs ``mpsylv.sylvester.bartels_stewart`` (pkg/src/mpsylv/sylvester.py:160-178) from
the read-only reference at /root/reference/pkg/src (build container only) on the
seeded config recipes at small sizes, plus the singular case that the reference's
triangular solve raises on (sylvester.py:141-143).  Re-run with

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_bs.py
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

from mpsylv.errors import SingularEquationError  # noqa: E402  (reference, read-only)
from mpsylv.sylvester import SylvesterProblem, bartels_stewart  # noqa: E402

from paper_2503_03456_b200 import problems  # noqa: E402

CASES = [  # tag, config recipe, m, n, seed
    ("c0", "c0", 24, 16, 0),
    ("c1", "c1", 20, 20, 1),
    ("c2", "c2", 24, 12, 2),
    ("c3", "c3", 16, 12, 3),
]


def main():
    out = {}
    for tag, cfg, m, n, seed in CASES:
        pr = problems.make(cfg, m, n, seed=seed)
        p = SylvesterProblem(pr.A, pr.B, pr.C, kind=pr.kind)
        t0 = time.time()
        X, rep = bartels_stewart(p)
        out[f"{tag}_A"], out[f"{tag}_B"], out[f"{tag}_C"] = pr.A, pr.B, pr.C
        out[f"{tag}_kind"] = np.array(pr.kind)
        out[f"{tag}_X"] = X
        out[f"{tag}_res"] = rep.residual
        print(f"{tag}: res={rep.residual:.2e} ({time.time() - t0:.1f}s)", flush=True)
    A = np.array([[1.0, 2.0], [0.0, 3.0]])
    B = np.array([[-1.0]])
    try:
        bartels_stewart(SylvesterProblem(A, B, np.ones((2, 1))))
        out["sing_rowcol"] = np.array([-1, -1])
    except SingularEquationError as e:
        out["sing_rowcol"] = np.array([e.row, e.col])
    out["sing_A"], out["sing_B"] = A, B
    np.savez_compressed(os.path.join(HERE, "bs.npz"), **out)


if __name__ == "__main__":
    main()
