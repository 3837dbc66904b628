"""Fingerprint scheme selection (reference `cache.py:26-91`, `kernels.py:114-120`).

Exact bit gathering ("precise mode") is used whenever the specification has at most 126 distinct
non-empty suffixes; otherwise the configured hash (MuellerHash by default, or the deliberately
weak first-k-positions scheme).  All variants then zero the lowest ``mask_bits`` bits.

Beyond the reference's domain (a characteristic matrix of more than 64 words: the reference refuses such
inputs, `enumerator.py:70-73`) the reference defines no hash.  There ``"mueller"`` resolves to this build's
NH fingerprint (`V_NH`; definition `oracle/ltl_oracle.c` fp_nh): two multiply-adds per word instead of
MuellerHash's four 64-bit multiplies, which is what bounds the screening kernel.  ``"mueller_blocked"``
keeps the blocked MuellerHash extension at every size, ``"nh"`` forces NH at every size (tests, A/B runs).
Inside the reference's domain ``"mueller"`` is the reference's MuellerHash bit for bit.

Whenever NH is selected and no trace has more than 32 positions, the variant is `V_NH32`: NH over row PAIRS
(definition `oracle/ltl_oracle.c` fp_nh32).  It goes with the device core's half-width store -- two rows per 64-bit
word, i.e. uint32 storage for L <= 32 (north-star subsystem 1): BASELINE config 4 moves 8 MiB instead of 16 MiB per matrix.
"""
from __future__ import annotations

from dataclasses import dataclass

FP_BITS = 126
V_GATHER, V_MUELLER, V_FKP, V_NH, V_NH32 = 0, 1, 2, 3, 4
HALF_WORD = 32  # rows of at most this many positions are stored two per 64-bit word
REFERENCE_WORDS = 64  # the reference's largest matrix: 64 rows x one word


@dataclass(frozen=True)
class HashScheme:
    variant: str = "mueller"  # "mueller" | "fkp" | "mueller_blocked" | "nh"
    mask_bits: int = 0

    def __post_init__(self):
        if self.variant not in ("mueller", "fkp", "mueller_blocked", "nh"):
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


def resolve_scheme(scheme: HashScheme, lengths, suffix_table=None, words_per_row: int = 1, *, n_rows: int | None = None,
                   max_len: int | None = None) -> ResolvedScheme:
    """``n_rows`` / ``max_len`` (with a suffix table): the two facts about the lengths the rule needs, for callers that
    hold them already (a device-resident specification) -- ``lengths`` is then not touched."""
    import numpy as np

    if suffix_table is not None and n_rows is not None and max_len is not None:
        lengths = None
    else:
        lengths = np.asarray(lengths, dtype=np.int64).reshape(-1)  # 2^21 traces: no per-element Python work below
        n_rows, max_len = len(lengths), (int(lengths.max()) if len(lengths) else 0)
    if suffix_table is not None:
        if suffix_table.count <= FP_BITS:
            return ResolvedScheme(V_GATHER, tuple(suffix_table.rows), tuple(suffix_table.offsets), mask_k=scheme.mask_bits)
    elif int(lengths.sum()) <= FP_BITS:
        rows = tuple(r for r, n in enumerate(lengths) for _ in range(int(n)))
        offs = tuple(j for n in lengths for j in range(int(n)))
        return ResolvedScheme(V_GATHER, rows, offs, mask_k=scheme.mask_bits)
    if scheme.variant in ("mueller", "mueller_blocked", "nh"):
        big = n_rows * int(words_per_row) > REFERENCE_WORDS
        nh = scheme.variant == "nh" or (scheme.variant == "mueller" and big)
        if nh and int(words_per_row) == 1 and max_len <= HALF_WORD:
            return ResolvedScheme(V_NH32, mask_k=scheme.mask_bits)
        return ResolvedScheme(V_NH if nh else V_MUELLER, mask_k=scheme.mask_bits)
    return ResolvedScheme(V_FKP, fkp_bits=fkp_bits_per_row(n_rows), mask_k=scheme.mask_bits)
