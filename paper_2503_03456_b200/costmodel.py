"""Leading-order flop counts of the paper's Table 3 (restated).

Same table as the reference's ``flops`` (pkg/src/mpsylv/costmodel.py:102-127;
PAPER.md:806-851).  Used to fill ``FlopCounter`` buckets and as the
algorithmic-flop definition of the bench roofline.
Complex problems are reported x4 by the bench (a complex multiply-add is 8
real flops against 2).
"""

from __future__ import annotations

from dataclasses import dataclass

ALGORITHMS = ("mp_orth_sylv", "mp_inv_sylv", "mp_orth_lyap", "mp_inv_lyap")


@dataclass(frozen=True)
class FlopCount:
    low_flops: float
    high_flops: float

    @property
    def total(self) -> float:
        return self.low_flops + self.high_flops


def flops(algorithm: str, m: int, n: int, k: int = 0) -> FlopCount:
    if k < 0:
        raise ValueError("k must be nonnegative")
    a = float(m ** 3 + n ** 3)
    b = float(m * n * (m + n))
    g = float(n ** 3)
    if algorithm == "mp_orth_sylv":
        return FlopCount(25.0 * a + b, 6.0 * a + (4.0 + 3.0 * k) * b)
    if algorithm == "mp_inv_sylv":
        return FlopCount(25.0 * a + b, (4.0 + 2.0 / 3.0) * a + (4.0 + 3.0 * k) * b)
    if algorithm == "mp_orth_lyap":
        return FlopCount(27.0 * g, (14.0 + 6.0 * k) * g)
    if algorithm == "mp_inv_lyap":
        return FlopCount(27.0 * g, (12.0 + 2.0 / 3.0 + 6.0 * k) * g)
    if algorithm == "bartels_stewart_sylv":
        return FlopCount(0.0, 25.0 * a + 5.0 * b)
    if algorithm == "bartels_stewart_lyap":
        return FlopCount(0.0, 35.0 * g)
    raise ValueError(f"unknown algorithm {algorithm!r}")


def algorithm_name(variant: str, kind: str) -> str:
    suffix = "lyap" if kind == "lyapunov" else "sylv"
    if variant == "bs":
        return f"bartels_stewart_{suffix}"
    return f"mp_{variant}_{suffix}"


def gemm_phase_flops(m: int, n: int, k: int, kind: str = "general") -> float:
    """fp64 GEMM-phase flops 6a + (4+2k)b, Sylvester form."""
    a = float(m ** 3 + n ** 3)
    b = float(m * n * (m + n))
    return 6.0 * a + (4.0 + 2.0 * k) * b
