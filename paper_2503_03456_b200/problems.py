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


# ---- the reference's ProblemGenerator kinds (cli.py:56-170), for harness and regime parity ----

KRON_CAP = 4096  # DEFAULT_KRON_CAP, linalg.py:66
_COND_CAP = {"normal": 6.0, "uniform": 15.0}  # transform condition caps (cli.py:104)
_ATTEMPTS = 400


@dataclass(frozen=True)
class ProblemGenerator:
    """Deterministic synthetic problem spec (cli.py:56-90): kinds random-dense,
    logspace-conditioned (eigenvalues 10^linspace(0, t)), hermitian, lyapunov."""

    kind: str
    m: int
    n: int
    t: float = 0.0
    seed: int = 0
    stream: int = 0

    def __post_init__(self):
        if self.kind not in ("random-dense", "logspace-conditioned", "hermitian", "lyapunov"):
            raise ValueError(f"unknown generator kind {self.kind!r}")
        if self.kind == "lyapunov" and self.m != self.n:
            raise ValueError("lyapunov generator requires m == n")
        if self.t < 0:
            raise ValueError("t must be nonnegative")


def _with_spectrum(P: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """P diag(lam) P^{-1}, the inverse applied as a solve with P^T (cli.py:97-100)."""
    return np.linalg.solve(P.T, (P * lam[None, :]).T).T


def _transform(rng, k: int, family: str) -> np.ndarray:
    """First draw whose 2-norm condition is under the family cap, else the best of the
    attempts (cli.py:107-119); every rejection consumes the same stream."""
    best, best_c = None, np.inf
    for _ in range(_ATTEMPTS):
        P = rng.standard_normal((k, k)) if family == "normal" else rng.random((k, k))
        c = np.linalg.cond(P)
        if c <= _COND_CAP[family]:
            return P
        if c < best_c:
            best, best_c = P, c
    return best


def _logspace(rng, m: int, n: int, t: float):
    """(A, B, C) with kappa_2(M_f) in [10^t, 10^(t+1)] while M_f is small enough to check
    (cli.py:122-143); otherwise the first draw."""
    checked = t >= 1.0 and m * n <= KRON_CAP
    best, best_d = None, np.inf
    for _ in range(_ATTEMPTS):
        A = _with_spectrum(_transform(rng, m, "normal"), np.logspace(0.0, t, m))
        B = _with_spectrum(_transform(rng, n, "uniform"), np.logspace(0.0, t, n))
        C = rng.standard_normal((m, n))
        if not checked:
            return A, B, C
        sv = np.linalg.svd(np.kron(np.eye(n), A) + np.kron(B.T, np.eye(m)), compute_uv=False)
        kap = float(sv[0] / sv[-1])
        if 10.0 ** t <= kap <= 10.0 ** (t + 1):
            return A, B, C
        d = abs(np.log10(kap) - (t + 0.5))
        if d < best_d:
            best, best_d = (A, B, C), d
    return best


def generate(g: ProblemGenerator) -> Problem:
    """The reference's generate() (cli.py:146-170) on the same Philox stream."""
    rng = rng_for(g.seed, g.stream)
    m, n = g.m, g.n
    if g.kind == "logspace-conditioned":
        A, B, C = _logspace(rng, m, n, g.t)
        return Problem(A, B, C, "general", "logspace", g.seed)
    if g.kind == "random-dense":
        A = rng.standard_normal((m, m))
        B = rng.standard_normal((n, n))
        return Problem(A, B, rng.standard_normal((m, n)), "general", "random-dense", g.seed)
    if g.kind == "hermitian":
        G = rng.standard_normal((m, m))
        A = (G + G.T) / 2 + (1.0 + np.sqrt(m)) * np.eye(m)
        G = rng.standard_normal((n, n))
        B = (G + G.T) / 2 + (1.0 + np.sqrt(n)) * np.eye(n)
        return Problem(A, B, rng.standard_normal((m, n)), "hermitian", "hermitian", g.seed)
    A = rng.standard_normal((m, m)) + (1.0 + np.sqrt(m)) * np.eye(m)
    G = rng.standard_normal((m, m))
    return Problem(A, A.conj().T, (G + G.T) / 2, "lyapunov", "lyapunov", g.seed)
