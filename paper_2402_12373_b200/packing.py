"""Trace packing into bit-sliced characteristic sequences (north-star subsystem 1, host side).

Layout (reference `bitsem.py:38-55`, `bitsem.py:73-88`, generalised by SURVEY rule N2 to W words
per row): position j of a trace lives in word ``j // 64`` at bit ``63 - j % 64`` (MSB first, so a
left shift moves position j+k to position j); bits at positions >= the trace length are 0.  One
characteristic matrix is ``uint64[R, W]`` with rows in specification order, positives first.

The reference packs with a Python triple loop (`bitsem.py:79-87`).  On the product path
(`TraceContext.from_spec(..., device=d)`, what `learn()` uses) the padded character matrix is packed by the
`k_pack` kernel of the CUDA library (`core.pack_traces`); without a device argument (host tools, workload
generators, tests that drive the learner with the CPU oracle) it is packed with `np.packbits`.  Same bits.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

WORD = 64


def words_for_length(max_len: int) -> int:
    return max(1, -(-int(max_len) // WORD))


def rounds_for_words(words: int) -> int:
    """ceil(log2(64*W)) shift rounds for F/G/U (reference `bitsem.py:39`, `bitsem.py:307-310`)."""
    r = 0
    while (1 << r) < WORD * words:
        r += 1
    return r


def _bits_to_words(bits: np.ndarray, W: int) -> np.ndarray:
    """bool[..., W*64] (position-major) -> uint64[..., W], position j at bit 63 - j%64."""
    packed = np.packbits(bits, axis=-1, bitorder="big")  # byte 0 holds positions 0..7, MSB first
    return packed.reshape(*bits.shape[:-1], W, 8).view(">u8").reshape(*bits.shape[:-1], W).astype(np.uint64)


def length_masks(lengths: np.ndarray, W: int) -> np.ndarray:
    """uint64[R, W]: ones at positions < length (reference `bitsem.py:51-55`)."""
    pos = np.arange(W * WORD)[None, :]
    return _bits_to_words(pos < np.asarray(lengths)[:, None], W)


@dataclass(frozen=True)
class TraceContext:
    """Per-specification packed data (reference `bitsem.py:64-101`)."""

    lengths: np.ndarray  # (R,) int64
    masks: np.ndarray  # (R, W) uint64
    n_pos: int
    atoms: np.ndarray  # (n_props, R, W) uint64
    words: int

    @staticmethod
    def from_spec(spec, alphabet, words: int | None = None, device: int | None = None) -> "TraceContext":
        W = words_for_length(spec.max_len) if words is None else int(words)
        if spec.max_len > W * WORD:
            raise ValueError(f"trace of length {spec.max_len} does not fit {W} word(s)")
        R, n_props = spec.size, alphabet.size
        if device is not None:
            from .core import pack_traces

            masks, atoms = pack_traces(spec.chars, spec.lengths, n_props, W, device)
            return TraceContext(spec.lengths.copy(), masks, spec.n_pos, atoms, W)
        chars = np.zeros((R, W * WORD), dtype=np.uint16)
        chars[:, : spec.chars.shape[1]] = spec.chars[:, : W * WORD]
        live = np.arange(W * WORD)[None, :] < spec.lengths[:, None]
        atoms = np.empty((n_props, R, W), dtype=np.uint64)
        for p in range(n_props):
            atoms[p] = _bits_to_words(((chars >> p) & 1).astype(bool) & live, W)
        return TraceContext(spec.lengths.copy(), _bits_to_words(live, W), spec.n_pos, atoms, W)

    @property
    def n_rows(self) -> int:
        return len(self.lengths)

    def atom_cm(self, prop: int) -> np.ndarray:
        return self.atoms[prop].copy()
