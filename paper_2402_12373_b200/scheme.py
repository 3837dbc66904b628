"""Fingerprint scheme selection (reference `cache.py:26-91`, `kernels.py:114-120`).

Exact bit gathering ("precise mode") is used whenever the specification has at most 126 distinct
non-empty suffixes; otherwise the configured hash (MuellerHash by default, or the deliberately
weak first-k-positions scheme).  All variants then zero the lowest ``mask_bits`` bits.
"""
from __future__ import annotations

from dataclasses import dataclass

FP_BITS = 126
V_GATHER, V_MUELLER, V_FKP = 0, 1, 2


@dataclass(frozen=True)
class HashScheme:
    variant: str = "mueller"  # "mueller" | "fkp"
    mask_bits: int = 0

    def __post_init__(self):
        if self.variant not in ("mueller", "fkp"):
            raise ValueError(f"unknown hash variant {self.variant!r}")
        if not 0 <= self.mask_bits <= FP_BITS:
            raise ValueError("mask_bits must lie in [0, 126]")


@dataclass(frozen=True)
class ResolvedScheme:
    variant: int
    proj_rows: tuple = ()
    proj_offs: tuple = ()
    fkp_bits: int = 0
    mask_k: int = 0

    @property
    def precise(self) -> bool:
        return self.variant == V_GATHER


def fkp_bits_per_row(n_rows: int) -> int:
    """Per-row prefix width bringing n_rows*width closest to 126 (reference `kernels.py:114-120`)."""
    lo = max(1, FP_BITS // n_rows)
    if abs((lo + 1) * n_rows - FP_BITS) < abs(lo * n_rows - FP_BITS):
        lo += 1
    return min(lo, 64)


def resolve_scheme(scheme: HashScheme, lengths, suffix_table=None) -> ResolvedScheme:
    if suffix_table is not None:
        if suffix_table.count <= FP_BITS:
            return ResolvedScheme(V_GATHER, tuple(suffix_table.rows), tuple(suffix_table.offsets), mask_k=scheme.mask_bits)
    elif sum(int(n) for n in lengths) <= FP_BITS:
        rows = tuple(r for r, n in enumerate(lengths) for _ in range(int(n)))
        offs = tuple(j for n in lengths for j in range(int(n)))
        return ResolvedScheme(V_GATHER, rows, offs, mask_k=scheme.mask_bits)
    if scheme.variant == "mueller":
        return ResolvedScheme(V_MUELLER, mask_k=scheme.mask_bits)
    return ResolvedScheme(V_FKP, fkp_bits=fkp_bits_per_row(len(lengths)), mask_k=scheme.mask_bits)
