"""Seeded synthetic problems for the five BASELINE configs (plus the headline CH).

Every generator draws float64 (or complex128) on the host with the
reference's own PRNG convention, ``Philox(SeedSequence(entropy=seed,
spawn_key=(stream,)))`` (reference ``pkg/src/mpsylv/cli.py:93-95``,
``GENERATOR_ID = "philox4x64-10"`` ``cli.py:54``).  The draw order is frozen
as in SURVEY.md section 8(d); identical arrays feed the oracle, the reference
and the GPU.  The paper's literature test set is not reproduced: these
seeded recipes stand in for it.

Arrays are returned in numpy C order (what the reference's
``SylvesterProblem`` holds); the GPU boundary converts to column-major.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GENERATOR_ID = "philox4x64-10"

CONFIGS = ("c0", "c1", "c2", "c3", "c4", "ch")

# full sizes of BASELINE.json's configs (SURVEY.md section 8 abbreviations)
FULL_SIZES = {
    "c0": (128, 128),
    "c1": (1024, 1024),
    "c2": (4096, 2048),
    "c3": (2048, 2048),
    "c4": (512, 512),
    "ch": (4096, 4096),
}


def rng_for(seed: int, stream: int = 0) -> np.random.Generator:
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(stream,))
    return np.random.Generator(np.random.Philox(ss))


@dataclass
class Problem:
    """A, B, C (numpy, C order) plus metadata; X_true only for c2."""

    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    kind: str = "general"
    config: str = ""
    seed: int = 0
    X_true: np.ndarray | None = None

    @property
    def m(self) -> int:
        return self.C.shape[0]

    @property
    def n(self) -> int:
        return self.C.shape[1]

    @property
    def is_complex(self) -> bool:
        return any(np.iscomplexobj(M) and np.any(np.imag(M) != 0)
                   for M in (self.A, self.B, self.C))


def _haar(rng, k):
    G = rng.standard_normal((k, k))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))[None, :]


def make_c0(m: int, n: int, seed: int = 0, stream: int = 0) -> Problem:
    """A = G_A/sqrt(m) + 2I, B = G_B/sqrt(n) + 2I, C ~ N(0,1)."""
    rng = rng_for(seed, stream)
    GA = rng.standard_normal((m, m))
    GB = rng.standard_normal((n, n))
    C = rng.standard_normal((m, n))
    A = GA / np.sqrt(m) + 2.0 * np.eye(m)
    B = GB / np.sqrt(n) + 2.0 * np.eye(n)
    return Problem(A, B, C, "general", "c0", seed)


def make_c1(n: int, seed: int = 0, stream: int = 0, rank: int = 16) -> Problem:
    """Lyapunov: A = G/sqrt(n) - 2.5I, B = A^T, C = -W W^T (W n x 16)."""
    rng = rng_for(seed, stream)
    G = rng.standard_normal((n, n))
    W = rng.standard_normal((n, rank))
    A = G / np.sqrt(n) - 2.5 * np.eye(n)
    C = -(W @ W.T)
    return Problem(A, A.T.copy(), C, "lyapunov", "c1", seed)


def make_c2(m: int, n: int, seed: int = 0, stream: int = 0) -> Problem:
    """Known solution: A = Q_A T_A Q_A^T, B = Q_B T_B Q_B^T, C = A X + X B."""
    rng = rng_for(seed, stream)
    dA = rng.uniform(1.0, 10.0, m)
    NA = rng.standard_normal((m, m)) * np.sqrt(0.25 / m)
    dB = rng.uniform(0.5, 5.0, n)
    NB = rng.standard_normal((n, n)) * np.sqrt(0.25 / n)
    QA = _haar(rng, m)
    QB = _haar(rng, n)
    X = rng.standard_normal((m, n))
    TA = np.diag(dA) + np.triu(NA, 1)
    TB = np.diag(dB) + np.triu(NB, 1)
    A = QA @ TA @ QA.T
    B = QB @ TB @ QB.T
    C = A @ X + X @ B
    return Problem(A, B, C, "general", "c2", seed, X_true=X)


def make_c3(m: int, n: int, seed: int = 0, stream: int = 0) -> Problem:
    """Complex: A = (G1+iG2)/sqrt(2m)+2I, B = (G3+iG4)/sqrt(2n)+(2+0.5i)I."""
    rng = rng_for(seed, stream)
    G1 = rng.standard_normal((m, m))
    G2 = rng.standard_normal((m, m))
    G3 = rng.standard_normal((n, n))
    G4 = rng.standard_normal((n, n))
    Cr = rng.standard_normal((m, n))
    Ci = rng.standard_normal((m, n))
    A = (G1 + 1j * G2) / np.sqrt(2 * m) + 2.0 * np.eye(m)
    B = (G3 + 1j * G4) / np.sqrt(2 * n) + (2.0 + 0.5j) * np.eye(n)
    C = (Cr + 1j * Ci) / np.sqrt(2.0)
    return Problem(A, B, C, "general", "c3", seed)


def make_c4(index: int, m: int = 512, seed: int = 0) -> Problem:
    """Equation ``index`` of the batch: the c0 recipe with entropy seed+index."""
    p = make_c0(m, m, seed + index, 0)
    p.config = "c4"
    return p


def make(config: str, m: int | None = None, n: int | None = None,
         seed: int = 0, stream: int = 0, index: int = 0) -> Problem:
    """Build one problem of ``config`` at full size or at (m, n)."""
    fm, fn = FULL_SIZES[config]
    m = fm if m is None else m
    n = (fn if config != "c0" and config != "ch" else m) if n is None else n
    if config in ("c0", "ch"):
        p = make_c0(m, n, seed, stream)
        p.config = config
        return p
    if config == "c1":
        return make_c1(m, seed, stream)
    if config == "c2":
        return make_c2(m, n, seed, stream)
    if config == "c3":
        return make_c3(m, n, seed, stream)
    if config == "c4":
        return make_c4(index, m, seed)
    raise ValueError(f"unknown config {config!r}")
