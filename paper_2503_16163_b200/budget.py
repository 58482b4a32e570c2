"""CacheBudget / memory_ratio -- same knobs and validation as the reference
(kvcache.py:23-63).  Pure host logic."""
from __future__ import annotations

import math
from dataclasses import dataclass
from decimal import ROUND_HALF_UP, Decimal

__all__ = ["CacheBudget", "memory_ratio", "FULL_PRECISION_BITS", "frontier"]

FULL_PRECISION_BITS = 16
_VALID_BITS = (1, 2, 4, FULL_PRECISION_BITS)


@dataclass(frozen=True)
class CacheBudget:
    """Knobs that determine the resident cache footprint (kvcache.py:29-52)."""

    bits: int = 2
    group_size: int = 32
    residual: int = 64
    prefetch_k: int = 64
    context_length: int = 4096

    def __post_init__(self) -> None:
        if self.bits not in _VALID_BITS:
            raise ValueError(f"bits must be one of {_VALID_BITS}")
        for name in ("group_size", "residual", "prefetch_k", "context_length"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    def ratio(self) -> float:
        return memory_ratio(self.bits, self.group_size, self.context_length,
                            self.residual + self.prefetch_k)


def memory_ratio(bits: int, group_size: float, context_length: int, resident_extra: int) -> float:
    """bits/16 + 2/g + (r+k)/L, half-up to 2 decimals (kvcache.py:55-63)."""
    raw = bits / 16.0 + (0.0 if math.isinf(group_size) else 2.0 / group_size)
    raw += resident_extra / context_length
    return float(Decimal(repr(raw)).quantize(Decimal("0.01"), rounding=ROUND_HALF_UP))


def frontier(n: int, residual: int, group: int) -> int:
    """Quantized frontier after n appends: g*floor((n-r)/g) for n >= r, else 0
    (the fixed point of the migrate-at-r+g loop, kvcache.py:169-171)."""
    return 0 if n < residual else group * ((n - residual) // group)
