"""Traces, specifications and the trace-file format (the input model either side of the hot path).

A trace is a sequence of characters; a character is an int bitmask over the alphabet's
propositions.  Contract follows the reference's `traces.py` (paths relative to
/root/reference/pkg/src/ltllearn/): `Alphabet` `traces.py:23-53`, `Specification`
`traces.py:56-106` (per-side de-duplication keeping first occurrences, P and N disjoint, row order
= positives then negatives), suffix table `traces.py:145-172`, file format `traces.py:180-253`.

Unlike the reference (tuples of tuples, <= 64 traces of <= 63 positions) a specification here is
backed by one padded ``uint16[R, Lmax]`` character matrix plus a length vector, so that 2^21
traces can be de-duplicated, censused and bit-packed with vectorised numpy / device code; the
tuple views `pos` / `neg` / `traces` are materialised lazily for small inputs.
"""
from __future__ import annotations

import warnings
from typing import Iterable, Sequence

import numpy as np

Trace = tuple


class TraceFormatError(ValueError):
    pass


class Alphabet:
    __slots__ = ("names",)

    def __init__(self, names: Sequence[str]):
        names = tuple(names)
        if not names:
            raise ValueError("alphabet must be non-empty")
        if len(set(names)) != len(names):
            raise ValueError("proposition names must be unique")
        for n in names:
            if n in ("X", "F", "G", "U") or not n or not all(c.isalnum() or c == "_" for c in n):
                raise ValueError(f"invalid proposition name {n!r}")
        object.__setattr__(self, "names", names)

    def __setattr__(self, *_):
        raise AttributeError("immutable")

    @staticmethod
    def default(size: int) -> "Alphabet":
        return Alphabet(tuple(f"p{i}" for i in range(size)))

    @property
    def size(self) -> int:
        return len(self.names)

    @property
    def n_chars(self) -> int:
        return 1 << len(self.names)

    def index_of(self, name: str):
        try:
            return self.names.index(name)
        except ValueError:
            return None

    def __eq__(self, other):
        return isinstance(other, Alphabet) and other.names == self.names

    def __hash__(self):
        return hash(self.names)

    def __repr__(self):
        return f"Alphabet({self.names})"


def _as_matrix(traces: Iterable) -> tuple[np.ndarray, np.ndarray]:
    rows = [np.asarray(tr, dtype=np.int64).reshape(-1) for tr in traces]
    lengths = np.array([len(r) for r in rows], dtype=np.int64)
    width = int(lengths.max()) if len(rows) else 0
    chars = np.zeros((len(rows), max(width, 1)), dtype=np.uint16)
    for k, r in enumerate(rows):
        if len(r):
            if r.min() < 0:
                raise ValueError("trace characters must be non-negative bitmasks")
            if r.max() > 0xFFFF:
                raise ValueError("at most 16 propositions are supported")
            chars[k, : len(r)] = r
    return chars, lengths


def _row_keys(chars: np.ndarray, lengths: np.ndarray, width: int) -> np.ndarray:
    """One opaque bytes-like key per trace: (length, padded characters)."""
    R = len(lengths)
    key = np.zeros((R, width + 1), dtype=np.uint16)
    key[:, 0] = lengths  # lengths < 65536 checked by callers
    key[:, 1 : 1 + chars.shape[1]] = chars
    return np.ascontiguousarray(key).view(np.dtype((np.void, key.dtype.itemsize * (width + 1)))).reshape(R)


def _first_occurrences(keys: np.ndarray) -> np.ndarray:
    _, first = np.unique(keys, return_index=True)
    return np.sort(first)


def _row_hashes(chars: np.ndarray, lengths: np.ndarray, width: int) -> np.ndarray:
    """64-bit hash of (length, padded characters) per trace, vectorised over the rows (a multilinear form over the
    row's 64-bit words, one pass).  Equal traces have equal hashes; unequal hashes prove traces different, so the
    exact (and slow: byte-string sort) comparison is only needed for the rare rows that share a hash."""
    R = len(lengths)
    if chars.shape[1] % 4 == 0 and chars.flags.c_contiguous and chars.dtype == np.uint16:
        words = chars.view(np.uint64)  # (R, width / 4), no copy
    else:
        cols = -(-max(chars.shape[1], 1) // 4) * 4
        key = np.zeros((R, cols), dtype=np.uint16)
        key[:, : chars.shape[1]] = chars
        words = key.view(np.uint64)
    k = np.arange(1, words.shape[1] + 1, dtype=np.uint64)
    consts = (k * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x632BE59BD9B4E019)) | np.uint64(1)
    h = words @ consts + lengths.astype(np.uint64) * np.uint64(0xD6E8FEB86659FD93)  # wraps mod 2^64
    h ^= h >> np.uint64(32)
    h *= np.uint64(0xBF58476D1CE4E5B9)
    h ^= h >> np.uint64(29)
    return h


def _member(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """a[i] in b, for uint64 hashes (sorted needles into a sorted haystack: np.isin is 10x slower on 10^6 keys)."""
    if len(b) == 0 or len(a) == 0:
        return np.zeros(len(a), dtype=bool)
    bs = np.sort(b)
    if len(b) > 4096:  # big haystack: walk it in order, then spread the few common values back
        a_s = np.sort(a)
        idx = np.minimum(np.searchsorted(bs, a_s), len(bs) - 1)
        common = np.unique(a_s[bs[idx] == a_s])
        if len(common) == 0:
            return np.zeros(len(a), dtype=bool)
        bs = common
    idx = np.minimum(np.searchsorted(bs, a), len(bs) - 1)
    return bs[idx] == a


def _dedup_first(chars: np.ndarray, lengths: np.ndarray, width: int):
    """Indices of the first occurrence of every distinct trace, ascending, and the row hashes."""
    h = _row_hashes(chars, lengths, width)
    hs = np.sort(h)
    dup_vals = hs[1:][hs[1:] == hs[:-1]]
    if len(dup_vals) == 0:
        return np.arange(len(lengths)), h
    suspects = np.flatnonzero(_member(h, dup_vals))  # ascending row indices
    keys = _row_keys(chars[suspects], lengths[suspects], width)
    first = suspects[_first_occurrences(keys)]
    drop = np.setdiff1d(suspects, first, assume_unique=True)
    keep = np.ones(len(lengths), dtype=bool)
    keep[drop] = False
    return np.flatnonzero(keep), h


class Specification:
    """Disjoint positive / negative trace sets in a fixed, meaningful order (it is the row order
    of every characteristic matrix: positives first)."""

    def __init__(self, pos=(), neg=(), *, _arrays=None):
        if _arrays is None:
            pc, pl = _as_matrix(pos)
            nc, nl = _as_matrix(neg)
        else:
            pc, pl, nc, nl = _arrays
        self._build(pc, pl, nc, nl)

    @staticmethod
    def from_arrays(pos_chars, pos_lengths, neg_chars, neg_lengths, *, device: int | None = None) -> "Specification":
        """Array form: ``chars[k, j]`` is character j of trace k (entries at j >= length ignored).

        ``device``: upload the character matrices to that GPU and do the specification's checks there
        (`core.DeviceTraces`: 128-bit row hashes filed with atomicMin screen for duplicate traces, the census of the
        overfit cost and the widest character are reduced on the device).  The host then touches the traces only if
        the device reports suspects -- duplicates or, with probability ~2^-128 per pair, a hash clash -- in which case
        the host path below decides (dropping duplicates with a warning, refusing traces on both sides) and the result
        is uploaded again.  `learn()` packs such a specification on the device and creates its core over the packed
        traces in place."""
        pl, nl = np.asarray(pos_lengths, dtype=np.int64).reshape(-1), np.asarray(neg_lengths, dtype=np.int64).reshape(-1)
        pc = np.ascontiguousarray(pos_chars, dtype=np.uint16).reshape(len(pl), -1)
        nc = np.ascontiguousarray(neg_chars, dtype=np.uint16).reshape(len(nl), -1)
        if device is None:
            return Specification(_arrays=(pc, pl, nc, nl))
        if max(int(pl.max()) if len(pl) else 0, int(nl.max()) if len(nl) else 0) > 0xFFFF:
            raise ValueError("traces longer than 65535 positions are not supported")
        from .core import DeviceTraces

        if len(pl) + len(nl) == 0:
            return Specification(_arrays=(pc, pl, nc, nl))
        dev = DeviceTraces(pc, pl, nc, nl, device)
        info = dev.info()
        if info["suspects"]:
            dev.close()
            spec = Specification(_arrays=(pc, pl, nc, nl))  # exact comparison, warnings, ValueError: the host rules
            if spec.size == 0:
                return spec
            dev = DeviceTraces(spec.chars[: spec.n_pos], spec.lengths[: spec.n_pos], spec.chars[spec.n_pos:],
                               spec.lengths[spec.n_pos:], device)
            info = dev.info()
            if info["suspects"]:  # pragma: no cover -- a 128-bit clash between different traces
                dev.close()
                return spec
            spec._attach(dev, info)
            return spec
        spec = Specification.__new__(Specification)
        spec.n_pos, spec.n_neg = len(pl), len(nl)
        spec._chars = spec._lengths = spec._tuples = None
        spec._sides = (pc, pl, nc, nl)
        spec._attach(dev, info)
        return spec

    def _attach(self, dev, info):
        self.device_traces, self._info = dev, info

    def release_device(self):
        """Free the device copy (it is also freed when the specification is collected)."""
        dev, self.device_traces = self.device_traces, None
        if dev is not None:
            dev.close()

    device_traces = None  # core.DeviceTraces when the specification is resident on a GPU
    _info = None          # its census (DeviceTraces.info())
    _sides = None         # device path: the caller's arrays, concatenated lazily into chars / lengths

    @property
    def chars(self) -> np.ndarray:
        """``uint16[R, Lmax]``, positives first, zero beyond each trace's length."""
        if self._chars is None:
            pc, pl, nc, nl = self._sides
            width = max(pc.shape[1] if len(pl) else 1, nc.shape[1] if len(nl) else 1, 1)
            full = np.zeros((len(pl) + len(nl), width), dtype=np.uint16)
            full[: len(pl), : pc.shape[1]] = pc
            full[len(pl):, : nc.shape[1]] = nc
            lengths = self.lengths
            if len(lengths) and int(lengths.min()) < width:
                full *= (np.arange(width)[None, :] < lengths[:, None]).astype(np.uint16)  # canonical zero padding
            self._chars = full
        return self._chars

    @property
    def lengths(self) -> np.ndarray:
        if self._lengths is None:
            _, pl, _, nl = self._sides
            self._lengths = np.concatenate([pl, nl]).astype(np.int64)
        return self._lengths

    def _build(self, pc, pl, nc, nl):
        width = max(pc.shape[1] if len(pl) else 1, nc.shape[1] if len(nl) else 1, 1)
        if max(int(pl.max()) if len(pl) else 0, int(nl.max()) if len(nl) else 0) > 0xFFFF:
            raise ValueError("traces longer than 65535 positions are not supported")

        def clean(chars, lengths):
            if len(lengths) and chars.shape[1] == width and int(lengths.min()) >= width:
                return np.ascontiguousarray(chars, dtype=np.uint16)  # every trace fills its row: nothing to pad
            full = np.zeros((len(lengths), width), dtype=np.uint16)
            if len(lengths):
                full[:, : chars.shape[1]] = chars
                full *= (np.arange(width)[None, :] < lengths[:, None]).astype(np.uint16)  # canonical zero padding
            return full

        pc, nc = clean(pc, pl), clean(nc, nl)
        sides = []
        for name, chars, lengths in (("positive", pc, pl), ("negative", nc, nl)):
            if len(lengths):
                keep, hashes = _dedup_first(chars, lengths, width)
                if len(keep) != len(lengths):
                    warnings.warn(f"{len(lengths) - len(keep)} duplicate {name} trace(s) dropped", stacklevel=4)
                    chars, lengths, hashes = chars[keep], lengths[keep], hashes[keep]
            else:
                hashes = np.zeros(0, dtype=np.uint64)
            sides.append((chars, lengths, hashes))
        (pc, pl, ph), (nc, nl, nh) = sides
        if len(ph) and len(nh):
            maybe = np.flatnonzero(_member(ph, nh))  # equal hashes: compare those few traces exactly
            if len(maybe):
                nsus = np.flatnonzero(_member(nh, ph[maybe]))
                pk, nk = _row_keys(pc[maybe], pl[maybe], width), _row_keys(nc[nsus], nl[nsus], width)
                clash = np.isin(pk, nk)
                if clash.any():
                    i = int(np.argmax(clash))
                    j = int(nsus[int(np.argmax(nk == pk[i]))])
                    raise ValueError(f"trace occurs on both sides (positive #{int(maybe[i])}, negative #{j})")
        self.n_pos = len(pl)
        self.n_neg = len(nl)
        self._chars = np.concatenate([pc, nc], axis=0) if (len(pl) + len(nl)) else np.zeros((0, width), np.uint16)
        self._lengths = np.concatenate([pl, nl]).astype(np.int64)
        self._tuples = None

    # -- views -------------------------------------------------------------------------
    @property
    def size(self) -> int:
        return self.n_pos + self.n_neg

    @property
    def max_len(self) -> int:
        if self._info is not None:
            return self._info["max_len"]
        return int(self.lengths.max()) if len(self.lengths) else 0

    @property
    def n_nonempty(self) -> int:
        return self._info["non_empty"] if self._info is not None else int(np.count_nonzero(self.lengths))

    @property
    def n_empty_positive(self) -> int:
        if self._info is not None:
            return self._info["empty_pos"]
        return int(np.count_nonzero(self.lengths[: self.n_pos] == 0))

    def _materialise(self):
        if self._tuples is None:
            self._tuples = tuple(
                tuple(int(c) for c in self.chars[r, : self.lengths[r]]) for r in range(self.size)
            )
        return self._tuples

    @property
    def traces(self) -> tuple:
        return self._materialise()

    @property
    def pos(self) -> tuple:
        return self._materialise()[: self.n_pos]

    @property
    def neg(self) -> tuple:
        return self._materialise()[self.n_pos :]

    def char_width(self) -> int:
        if self._info is not None:
            return max(1, self._info["char_or"].bit_length())
        top = int(np.bitwise_or.reduce(self.chars, axis=None)) if self.chars.size else 0
        return max(1, top.bit_length())

    def positive_char_census(self) -> tuple[int, int]:
        """(#positions, #set proposition bits) over the positive traces -- all that the
        closed-form overfit cost needs."""
        if self._info is not None:
            return self._info["pos_positions"], self._info["pos_bits"]
        pc = self.chars[: self.n_pos]
        n_positions = int(self.lengths[: self.n_pos].sum())
        # padding beyond each length is canonical zero, so the set bits of the whole matrix are the census
        return n_positions, int(np.bitwise_count(pc).sum(dtype=np.int64))

    def __repr__(self):
        return f"Specification(|P|={self.n_pos}, |N|={self.n_neg}, max_len={self.max_len})"


# ---------------------------------------------------------------------------------- suffix table


class SuffixTable:
    """One representative (row, offset) per distinct non-empty suffix, in first-occurrence scan
    order (row-major).  Only its size decides whether fingerprints can be exact (<= 126), so the
    scan stops as soon as ``limit`` distinct suffixes have been seen: ``count`` is then
    ``limit + 1`` ("too many") and the projection is meaningless.  (Reference `traces.py:145-172`
    scans everything, O(R*L^2); every non-empty trace is its own suffix, so R > limit + 1 traces
    already decide the question.)"""

    __slots__ = ("count", "rows", "offsets", "complete")

    def __init__(self, count, rows, offsets, complete):
        self.count, self.rows, self.offsets, self.complete = count, tuple(rows), tuple(offsets), complete

    @staticmethod
    def from_spec(spec: Specification, limit: int | None = None) -> "SuffixTable":
        if limit is not None and spec.n_nonempty > limit:
            return SuffixTable(limit + 1, (), (), False)
        seen = set()
        rows, offs = [], []
        for r, tr in enumerate(spec.traces):
            for j in range(len(tr)):
                suf = tr[j:]
                if suf not in seen:
                    seen.add(suf)
                    rows.append(r)
                    offs.append(j)
                    if limit is not None and len(seen) > limit:
                        return SuffixTable(limit + 1, (), (), False)
        return SuffixTable(len(seen), rows, offs, True)


# ---------------------------------------------------------------------------------- file format
# One trace per line, positions separated by ';', each position a comma-separated 0/1 vector
# over the alphabet; a '---' line separates positives from negatives; later sections ignored.


def _parse_line(line: str, line_no: int, width):
    chars = []
    for token in line.split(";"):
        bits = token.split(",")
        if width is None:
            width = len(bits)
        elif len(bits) != width:
            raise TraceFormatError(f"line {line_no}: expected {width} propositions, found {len(bits)}")
        char = 0
        for p, b in enumerate(bits):
            b = b.strip()
            if b == "1":
                char |= 1 << p
            elif b != "0":
                raise TraceFormatError(f"line {line_no}: bad proposition value {b!r}")
        chars.append(char)
    return tuple(chars), width


def _load_spec_lines(path) -> tuple[Specification, Alphabet]:
    """Line-by-line parser: the reference's reader (`traces.py:185-253`), with its error messages."""
    sections: list[list] = [[]]
    width = None
    with open(path, "r", encoding="utf-8") as fh:
        for line_no, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line:
                continue
            if line == "---":
                sections.append([])
                continue
            tr, width = _parse_line(line, line_no, width)
            sections[-1].append(tr)
    if len(sections) < 2:
        raise TraceFormatError("missing '---' separator between trace blocks")
    if len(sections) > 2:
        warnings.warn(f"{path}: ignoring {len(sections) - 2} extra '---' section(s)")
    if width is None:
        raise TraceFormatError("empty trace file")
    return Specification(tuple(sections[0]), tuple(sections[1])), Alphabet.default(width)


def _load_spec_arrays(data: bytes):
    """Whole-file parser for files in canonical form (only the bytes ``0 1 , ; -`` and line ends): every step is one
    numpy pass over the file, so 2^21 traces parse in seconds instead of minutes.  Returns ``(pc, pl, nc, nl, width,
    extra_sections)`` or None when the file needs the line-by-line reader (other bytes, malformed lines: that reader owns
    the error messages)."""
    b = np.frombuffer(data, dtype=np.uint8)
    if len(b) == 0:
        return None
    if b[-1] != 10:
        b = np.concatenate([b, np.array([10], dtype=np.uint8)])
    is_nl, is_cr = b == 10, b == 13
    is_d = (b == 48) | (b == 49)
    is_c, is_s, is_m = b == 44, b == 59, b == 45
    if not (is_nl | is_cr | is_d | is_c | is_s | is_m).all():
        return None
    line_of = np.cumsum(is_nl) - is_nl  # line index of every byte (the newline belongs to its line)
    n_lines = int(line_of[-1]) + 1

    def per_line(mask):
        return np.bincount(line_of[mask], minlength=n_lines)

    n_d, n_c, n_s, n_m = per_line(is_d), per_line(is_c), per_line(is_s), per_line(is_m)
    blank = (n_d + n_c + n_s + n_m) == 0
    sep = (n_m == 3) & (n_d + n_c + n_s == 0)
    if ((n_m > 0) & ~sep).any():
        return None
    trace = ~blank & ~sep
    if not trace.any():
        return None
    first = int(np.flatnonzero(trace)[0])
    n_pos_first = int(n_s[first]) + 1
    if n_d[first] % n_pos_first:
        return None
    width = int(n_d[first]) // n_pos_first
    if width < 1 or width > 16:
        return None
    n_positions = n_s + 1
    ok = (n_d == n_positions * width) & (n_c == n_positions * (width - 1))
    if not ok[trace].all():
        return None
    # token structure: between two digits of a line sits exactly one separator (so no "01", ",," or ";," forms)
    body = ~(is_nl | is_cr | is_m)
    prev_is_d = np.concatenate([[False], is_d[:-1]])
    prev_is_body = np.concatenate([[False], body[:-1]])
    if (is_d & prev_is_d).any() or ((is_c | is_s) & ~prev_is_d).any():
        return None
    line_end_sep = is_nl & np.concatenate([[False], (is_c | is_s)[:-1]])  # a line must not end in a separator
    if line_end_sep.any():
        return None
    del prev_is_body
    # digit k of a line is proposition k % width of position k // width
    d_idx = np.flatnonzero(is_d)
    d_line = line_of[d_idx]
    first_digit = np.zeros(n_lines, dtype=np.int64)
    first_digit[1:] = np.cumsum(n_d)[:-1]
    k = np.arange(len(d_idx), dtype=np.int64) - first_digit[d_line]
    ones = b[d_idx] == 49
    # separators must alternate correctly: the separator before digit k > 0 is ';' iff k % width == 0
    sep_before = np.zeros(len(d_idx), dtype=np.uint8)
    has_prev = k > 0
    sep_before[has_prev] = b[d_idx[has_prev] - 1]
    if ((sep_before[has_prev] == 59) != (k[has_prev] % width == 0)).any():
        return None
    section = np.cumsum(sep)[trace]  # section index of every trace line
    t_lines = np.flatnonzero(trace)
    t_index = np.full(n_lines, -1, dtype=np.int64)
    t_index[t_lines] = np.arange(len(t_lines))
    lengths = n_positions[t_lines].astype(np.int64)
    L = int(lengths.max())
    rows = t_index[d_line[ones]]
    kk = k[ones]
    flat = np.bincount(rows * L + kk // width, weights=(1 << (kk % width)).astype(np.float64), minlength=len(t_lines) * L)
    chars = flat.astype(np.uint16).reshape(len(t_lines), L)
    p_sel, n_sel = section == 0, section == 1
    return chars[p_sel], lengths[p_sel], chars[n_sel], lengths[n_sel], width, int(sep.sum()) - 1


def load_spec(path, *, device: int | None = None) -> tuple[Specification, Alphabet]:
    """Read a trace file (reference `traces.py:185-253`).  Big files in canonical form are parsed by the library's two-pass
    byte reader (`core.parse_trace_file`; 2^21 traces: about a second), or with whole-file numpy passes when the library
    is not built (`_load_spec_arrays`); anything else -- and every malformed file -- goes through the reference's line-by-line reader,
    which owns the error messages.  ``device``: keep the specification resident on that GPU (`from_arrays`)."""
    with open(path, "rb") as fh:
        data = fh.read()
    got = None
    if len(data) > (1 << 14) or device is not None:
        try:  # the library's two-pass byte reader (host code); without the library: the numpy passes
            from .core import parse_trace_file

            got = parse_trace_file(data)
        except Exception:  # noqa: BLE001 -- e.g. the library is not built
            got = _load_spec_arrays(data)
    if got is None:
        return _load_spec_lines(path)
    pc, pl, nc, nl, width, extra = got
    if extra < 0:
        raise TraceFormatError("missing '---' separator between trace blocks")
    if extra > 0:
        warnings.warn(f"{path}: ignoring {extra} extra '---' section(s)")
    return Specification.from_arrays(pc, pl, nc, nl, device=device), Alphabet.default(width)


def format_trace(tr, width: int) -> str:
    return ";".join(",".join("1" if (int(c) >> p) & 1 else "0" for p in range(width)) for c in tr)


def save_spec(spec: Specification, path, alphabet: Alphabet | None = None) -> None:
    width = alphabet.size if alphabet is not None else spec.char_width()
    if (spec.lengths == 0).any():
        raise TraceFormatError("the trace file format cannot carry empty traces")
    with open(path, "w", encoding="utf-8") as fh:
        for tr in spec.pos:
            fh.write(format_trace(tr, width) + "\n")
        fh.write("---\n")
        for tr in spec.neg:
            fh.write(format_trace(tr, width) + "\n")
