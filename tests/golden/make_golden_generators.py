"""Pin the problem generators against the REFERENCE's own (cli.py:56-170).

Runs the read-only reference ``mpsylv.cli.generate`` for a set of generator specs and
stores SHA-256 digests of the (A, B, C) arrays it returns; tests/test_host.py checks that
paper_2503_03456_b200.problems.generate reproduces them byte for byte.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_generators.py
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from mpsylv.cli import ProblemGenerator, generate  # noqa: E402  (reference, read-only)

SPECS = [
    ("logspace-conditioned", 10, 10, 2.0, 7, 0),
    ("logspace-conditioned", 10, 10, 12.0, 7, 0),
    ("logspace-conditioned", 8, 8, 3.0, 11, 0),
    ("logspace-conditioned", 9, 7, 5.0, 31, 17),
    ("logspace-conditioned", 72, 72, 4.0, 1, 3),
    ("random-dense", 5, 4, 0.0, 3, 1),
    ("hermitian", 6, 5, 0.0, 2, 0),
    ("lyapunov", 6, 6, 0.0, 2, 4),
]


def digest(M) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(M, dtype=np.complex128)).tobytes()).hexdigest()


def main():
    out = []
    for spec in SPECS:
        p = generate(ProblemGenerator(*spec))
        out.append({"spec": list(spec), "kind": p.kind, "A": digest(p.A), "B": digest(p.B), "C": digest(p.C)})
    with open(os.path.join(HERE, "generators.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out), "specs")


if __name__ == "__main__":
    main()
