"""Precision descriptors and flop accounting (boundary types of the hot path).

Mirrors the data types of ``mpsylv.precision`` that appear in the solver
signatures (pkg/src/mpsylv/precision.py:61-172): ``FpFormat`` and the six
predefined formats, ``FlopCounter`` and ``PrecisionContext``.  The rounding
simulator itself is deliberately absent: the device computes in IEEE
binary32 / binary64 hardware arithmetic.
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class FpFormat:
    name: str
    significand_bits: int
    exponent_bits: int
    supports_subnormals: bool = True

    @property
    def unit_roundoff(self) -> float:
        return 2.0 ** -self.significand_bits

    @property
    def is_binary64(self) -> bool:
        return self.significand_bits == 53 and self.exponent_bits == 11

    @property
    def is_binary32(self) -> bool:
        return self.significand_bits == 24 and self.exponent_bits == 8

    @classmethod
    def from_bits(cls, significand_bits: int, exponent_bits: int, name: str | None = None) -> "FpFormat":
        return cls(name or f"p{significand_bits}e{exponent_bits}", significand_bits, exponent_bits)


BFLOAT16 = FpFormat("bfloat16", 8, 8)
BINARY16 = FpFormat("binary16", 11, 5)
TF32 = FpFormat("tf32", 11, 8)
B24 = FpFormat("b24", 16, 8)
BINARY32 = FpFormat("binary32", 24, 8)
BINARY64 = FpFormat("binary64", 53, 11)

FORMATS = {f.name: f for f in (BFLOAT16, BINARY16, TF32, B24, BINARY32, BINARY64)}


def format_from_name(name: str) -> FpFormat:
    try:
        return FORMATS[name.lower()]
    except KeyError:
        raise ValueError(f"unknown format {name!r}; known: {sorted(FORMATS)}") from None


def parse_format(spec: str) -> FpFormat:
    if ":" in spec:
        t, e = spec.split(":", 1)
        return FpFormat.from_bits(int(t), int(e))
    return format_from_name(spec)


def format_bits(fmt) -> int:
    """32 or 64 for the two hardware formats (duck-typed on the reference's FpFormat too)."""
    t, e = int(fmt.significand_bits), int(fmt.exponent_bits)
    if (t, e) == (24, 8):
        return 32
    if (t, e) == (53, 11):
        return 64
    return 0


class FlopCounter:
    """Accumulates operation counts into named buckets (precision.py:148-172).

    The drop-in fills it from the paper's flop model (costmodel.flops), not
    by counting scalar operations; see ``refinement.mp_orth``.
    """

    def __init__(self):
        self.counts: dict[str, int] = {}

    def add(self, bucket: str, n: int) -> None:
        self.counts[bucket] = self.counts.get(bucket, 0) + int(n)

    def get(self, bucket: str) -> int:
        return self.counts.get(bucket, 0)

    def total(self) -> int:
        return sum(self.counts.values())

    def reset(self) -> None:
        self.counts.clear()

    def __repr__(self):
        inner = ", ".join(f"{k}={v}" for k, v in sorted(self.counts.items()))
        return f"FlopCounter({inner})"


@dataclass(frozen=True)
class PrecisionContext:
    format: FpFormat
    counter: FlopCounter | None = field(default=None, compare=False)
    bucket: str = "high"

    @property
    def unit_roundoff(self) -> float:
        return self.format.unit_roundoff

    def count(self, n: int) -> None:
        if self.counter is not None:
            self.counter.add(self.bucket, n)
