"""Bottom-up, cost-increasing search for a minimal separating LTL formula -- host-side level driver.

This is the caller of the hot path: it packs the specification, seeds the language cache with the
atoms, and for every cost level hands the device core the ordered list of candidate *segments*
(`(op, left bucket range, right bucket range, triangular)`), which the core screens in one pass
per level (evaluate -> P/N check -> fingerprint -> dedup -> append).  Behaviour follows the
reference's `enumerator.py` (paths relative to /root/reference/pkg/src/ltllearn/): validation
`enumerator.py:129-140`, atom fast path `182-192`, cache init `218-232`, level loop `234-251`,
child-cost pairing `254-268`, dispatch order `271-296`.  Differences by design: no 64-trace /
63-position limit (rows and words per row are free parameters of the device core), and one
`run_level` call per cost level instead of one Python call per 2^22-candidate chunk.

There is no CPU fallback: without the CUDA library `make_core` raises `BackendUnavailable`.
Tests inject other cores (the CPU oracle) through ``core_factory``.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, NamedTuple, Optional, Sequence, Union

import numpy as np

from .cache import LanguageCache
from .errors import CoreOOM, TimeoutExceeded
from .formula import (
    COMMUTATIVE_OPS,
    CONNECTIVE_ORDER,
    OP_ATOM,
    OP_NOT,
    OP_UNTIL,
    UNARY_OPS,
    UNIFORM,
    Atom,
    CostHomomorphism,
    Formula,
    Not,
    overfit,
    overfit_cost,
    print_formula,
)
from .packing import TraceContext
from .scheme import HashScheme, resolve_scheme
from .traces import Alphabet, Specification, SuffixTable

S_DONE, S_SOLVED, S_OOM, S_TIMEOUT = 0, 1, 2, 3
MAX_WORDS_PER_ROW = 16  # device kernels are instantiated for rows of up to 1024 positions


class Segment(NamedTuple):
    """One run of candidates in enumeration order: ``op`` applied to left entries [a0, a1) and,
    for binary ops, right entries [b0, b1); ``tri`` restricts to right index > left index."""

    op: int
    a0: int
    a1: int
    b0: int = -1
    b1: int = -1
    tri: bool = False

    @property
    def unary(self) -> bool:
        return self.b0 < 0


@dataclass
class LearnerConfig:
    cost: CostHomomorphism = UNIFORM
    require_nnf: bool = False
    forbid_until: bool = False
    hash: HashScheme = field(default_factory=HashScheme)
    budget_bytes: int = 2 << 30  # logical budget, admitted * (8*R*W + 16) (reference `_speedups.pyx:100`)
    noise: float = 0.0
    ceiling: Optional[int] = None  # exclusive: levels run up to ceiling - 1
    deadline: Optional[float] = None  # time.monotonic() cutoff
    device: int = 0
    max_traces: Optional[int] = None
    max_trace_len: int = MAX_WORDS_PER_ROW * 64
    #: keep the characteristic matrices of the last cost level too.  They are never operands (the search
    #: ends there), so by default only their fingerprints and records are kept; results are identical.
    store_last_level: bool = False
    #: pack the traces with the CUDA library's k_pack (None: yes unless a core factory is injected)
    pack_on_device: Optional[bool] = None

    def __post_init__(self):
        if not 0.0 <= self.noise <= 1.0:
            raise ValueError("noise must lie in [0, 1]")
        if self.max_trace_len < 1 or self.max_trace_len > MAX_WORDS_PER_ROW * 64:
            raise ValueError(f"max_trace_len must lie in [1, {MAX_WORDS_PER_ROW * 64}]")

    def err_max(self, spec: Specification) -> int:
        return math.floor(self.noise * spec.size + 1e-9)


@dataclass
class EnumStats:
    offered: int = 0
    admitted: int = 0
    duplicates: int = 0
    peak_bytes: int = 0
    precise: bool = False
    ceiling: int = 0
    atom_fast_path: bool = False
    levels: list = field(default_factory=list)
    search_seconds: float = 0.0
    h2d_bytes: int = 0  # host->device / device->host bytes moved by the device core for this search
    d2h_bytes: int = 0
    phase_ms: dict = field(default_factory=dict)  # host wall time of the call's phases (pack, scheme, create, close)

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("offered", "admitted", "duplicates", "peak_bytes", "precise",
                                              "ceiling", "atom_fast_path", "levels")}


@dataclass
class Solved:
    formula: Formula
    cost: int
    stats: EnumStats


@dataclass
class OutOfMemory:
    stats: EnumStats


class CeilingReached:
    """No separating formula below the ceiling; ``formula`` is the overfitting formula, which always
    separates (built lazily: for 2^20 positive traces the tree itself is enormous)."""

    def __init__(self, spec, alphabet, ceiling: int, stats: EnumStats):
        self._spec, self._alphabet = spec, alphabet
        self.ceiling, self.stats = ceiling, stats
        self._formula = None

    @property
    def formula(self) -> Formula:
        if self._formula is None:
            self._formula = overfit(self._spec, self._alphabet)
        return self._formula


EnumOutcome = Union[Solved, OutOfMemory, CeilingReached]


def _validate(spec: Specification, alphabet: Alphabet, cfg: LearnerConfig):
    if not spec.n_pos or not spec.n_neg:
        raise ValueError("need at least one positive and one negative trace")
    if cfg.max_traces is not None and spec.size > cfg.max_traces:
        raise ValueError(f"{spec.size} traces exceed the limit of {cfg.max_traces}")
    if spec.max_len > cfg.max_trace_len:
        raise ValueError(f"trace of length {spec.max_len} exceeds {cfg.max_trace_len}")
    if spec.n_empty_positive:
        raise ValueError("an empty positive trace can never be satisfied")
    if spec.char_width() > alphabet.size:
        raise ValueError("traces use propositions outside the alphabet")


def enabled_ops(cfg: LearnerConfig) -> list[int]:
    return [op for op in CONNECTIVE_ORDER
            if not (op == OP_NOT and cfg.require_nnf) and not (op == OP_UNTIL and cfg.forbid_until)]


def bucket_pairs(cost: CostHomomorphism, c: int, op: int):
    """Child-cost combinations for cost-c candidates with top connective op (reference
    `enumerator.py:254-268`)."""
    w = cost.of(op)
    if op in UNARY_OPS:
        return [(c - w, None)] if c - w >= 1 else []
    pairs = []
    for a in range(1, c - w):
        b = c - w - a
        if b < 1:
            continue
        if op in COMMUTATIVE_OPS and a > b:
            break
        pairs.append((a, b))
    return pairs


def level_segments(cache: LanguageCache, cfg: LearnerConfig, ops: Sequence[int], c: int) -> list[Segment]:
    """The level's candidates as ordered segments (dispatch order of reference
    `enumerator.py:271-296`; empty segments dropped)."""
    segs = []
    for op in ops:
        for a, b in bucket_pairs(cfg.cost, c, op):
            sa, ea = cache.bucket_range(a)
            if b is None:
                if ea > sa:
                    segs.append(Segment(op, sa, ea))
                continue
            sb, eb = cache.bucket_range(b)
            if ea == sa or eb == sb:
                continue
            segs.append(Segment(op, sa, ea, sb, eb, op in COMMUTATIVE_OPS and a == b))
    return segs


def _host_error_count(cm: np.ndarray, n_pos: int) -> int:
    """Rows whose position-0 verdict disagrees with their side (reference `bitsem.py:157-160`);
    used only for the bare-atom fast path before any core exists."""
    bit0 = (cm[:, 0] >> np.uint64(63)).astype(bool)
    return int(np.count_nonzero(~bit0[:n_pos])) + int(np.count_nonzero(bit0[n_pos:]))


def _check_deadline(cfg: LearnerConfig):
    if cfg.deadline is not None and time.monotonic() > cfg.deadline:
        raise TimeoutExceeded("learner deadline exceeded")


def _run_level(core, segs: list[Segment], cfg: LearnerConfig):
    """(status, op, li, ri) of the first non-DONE event, or None."""
    if hasattr(core, "run_level"):
        if cfg.deadline is not None and hasattr(core, "set_option"):
            # the level is one call: the core checks the deadline between its passes, as the reference does between its
            # 2^22-candidate chunks (`enumerator.py:278`, `290`)
            core.set_option("deadline_ms", max(1, int(1e3 * (cfg.deadline - time.monotonic()))))
        status, k, li, ri = core.run_level(segs)
        if status == S_TIMEOUT:
            raise TimeoutExceeded("learner deadline exceeded")
        return None if status == S_DONE else (status, segs[k].op if k >= 0 else -1, li, ri)
    for s in segs:
        _check_deadline(cfg)
        if s.unary:
            status, li, ri = core.screen_unary(s.op, s.a0, s.a1)
        else:
            status, li, ri = core.screen_binary(s.op, s.a0, s.a1, s.b0, s.b1, s.tri)
        if status != S_DONE:
            return status, s.op, li, ri
    return None


class Enumeration:
    """One bottom-up search, split into `__init__` (validate, pack, atom fast path, create the device core,
    admit the atoms -- everything up to "inputs resident in HBM") and `run` (the cost-level loop)."""

    def __init__(self, spec: Specification, alphabet: Alphabet, cfg: LearnerConfig | None = None, *,
                 core_factory: Callable | None = None):
        cfg = cfg or LearnerConfig()
        _validate(spec, alphabet, cfg)
        self.spec, self.alphabet, self.cfg = spec, alphabet, cfg
        # product path (no injected core): packing runs on the device too; an injected core factory (tests with
        # the CPU oracle, the sharded wrapper) gets host-packed inputs
        on_device = cfg.pack_on_device if cfg.pack_on_device is not None else core_factory is None
        self.stats = stats = EnumStats()
        self.outcome: EnumOutcome | None = None
        self.core = None
        self.cache = None
        self._traces = None
        dev = spec.device_traces
        if dev is not None and core_factory is None and dev.device_index == cfg.device:
            self._init_resident(dev)  # the specification is in HBM already: nothing but counters crosses the host
            return
        t_pack = time.perf_counter()
        self.ctx = ctx = TraceContext.from_spec(spec, alphabet, device=cfg.device if on_device else None)
        n_pos, err_max, h = spec.n_pos, cfg.err_max(spec), cfg.cost
        stats.phase_ms["pack"] = 1e3 * (time.perf_counter() - t_pack)
        stats.ceiling = overfit_cost(spec, alphabet, h)
        self.ceiling = stats.ceiling if cfg.ceiling is None else min(cfg.ceiling, stats.ceiling)

        atom_c = h.of(OP_ATOM)
        for p in range(alphabet.size):
            if _host_error_count(ctx.atoms[p], n_pos) <= err_max:
                stats.atom_fast_path = True
                self.outcome = Solved(Atom(p), atom_c, stats)
                return
        if cfg.require_nnf:
            for p in range(alphabet.size):
                if _host_error_count(~ctx.atoms[p] & ctx.masks, n_pos) <= err_max:
                    stats.atom_fast_path = True
                    self.outcome = Solved(Not(Atom(p)), atom_c + h.of(OP_NOT), stats)
                    return

        t_scheme = time.perf_counter()
        rs = resolve_scheme(cfg.hash, ctx.lengths, SuffixTable.from_spec(spec, limit=126), words_per_row=ctx.words)
        stats.precise = rs.precise
        t_create = time.perf_counter()
        stats.phase_ms["scheme"] = 1e3 * (t_create - t_scheme)
        if core_factory is None:
            from .core import make_core as core_factory  # CUDA core; raises BackendUnavailable
        self.core = core_factory(ctx.masks, n_pos, err_max, rs.variant, rs.proj_rows, rs.proj_offs, rs.fkp_bits,
                                 rs.mask_k, cfg.budget_bytes, words_per_row=ctx.words, device=cfg.device)
        self.cache = cache = LanguageCache(self.core)
        self._t_search = time.perf_counter()
        stats.phase_ms["create"] = 1e3 * (self._t_search - t_create)
        try:
            admitted_atoms = [p for p in range(alphabet.size)
                              if cache.try_admit(ctx.atoms[p], (OP_ATOM, p, -1), atom_c)]
            if cfg.require_nnf:
                neg_c = atom_c + h.of(OP_NOT)
                for entry, p in enumerate(admitted_atoms):
                    cache.try_admit(~ctx.atoms[p] & ctx.masks, (OP_NOT, entry, -1), neg_c)
        except CoreOOM:
            self.outcome = self._finish(OutOfMemory(stats))

    def _init_resident(self, dev):
        """`__init__` for a device-resident specification (`Specification.from_arrays(..., device=d)`): packing
        (`bitsem.py:73-88`), the atom fast path (`enumerator.py:182-192`) and the admission of the atoms (`218-232`) run on
        the device over the uploaded character matrix; masks and atoms never visit the host."""
        spec, alphabet, cfg, stats = self.spec, self.alphabet, self.cfg, self.stats
        err_max, h = cfg.err_max(spec), cfg.cost
        t_pack = time.perf_counter()
        dev.pack(alphabet.size)
        info = dev.info()
        self.ctx = None
        self._traces = dev
        stats.phase_ms["pack"] = 1e3 * (time.perf_counter() - t_pack)
        stats.ceiling = overfit_cost(spec, alphabet, h)
        self.ceiling = stats.ceiling if cfg.ceiling is None else min(cfg.ceiling, stats.ceiling)
        atom_c = h.of(OP_ATOM)
        fast = None
        for p in range(alphabet.size):
            if info["atom_errors"][p] <= err_max:
                fast = Solved(Atom(p), atom_c, stats)
                break
        if fast is None and cfg.require_nnf:
            for p in range(alphabet.size):
                if info["neg_atom_errors"][p] <= err_max:
                    fast = Solved(Not(Atom(p)), atom_c + h.of(OP_NOT), stats)
                    break
        if fast is not None:
            stats.atom_fast_path = True
            stats.h2d_bytes, stats.d2h_bytes = info["h2d_bytes"], info["d2h_bytes"]  # the upload is all this search moved
            self.outcome = fast
            return
        t_scheme = time.perf_counter()
        words = info["words"]
        rs = resolve_scheme(cfg.hash, None, SuffixTable.from_spec(spec, limit=126), words_per_row=words, n_rows=spec.size,
                            max_len=info["max_len"])
        stats.precise = rs.precise
        t_create = time.perf_counter()
        stats.phase_ms["scheme"] = 1e3 * (t_create - t_scheme)
        from .core import make_core

        self.core = make_core(None, spec.n_pos, err_max, rs.variant, rs.proj_rows, rs.proj_offs, rs.fkp_bits, rs.mask_k,
                              cfg.budget_bytes, words_per_row=words, device=cfg.device, traces=dev)
        self.cache = cache = LanguageCache(self.core)
        self._t_search = time.perf_counter()
        stats.phase_ms["create"] = 1e3 * (self._t_search - t_create)
        try:
            admitted_atoms = [p for p in range(alphabet.size)
                              if cache.try_admit_atom(dev, p, False, (OP_ATOM, p, -1), atom_c)]
            if cfg.require_nnf:
                neg_c = atom_c + h.of(OP_NOT)
                for entry, p in enumerate(admitted_atoms):
                    cache.try_admit_atom(dev, p, True, (OP_NOT, entry, -1), neg_c)
        except CoreOOM:
            self.outcome = self._finish(OutOfMemory(stats))

    def _finish(self, outcome):
        core, stats = self.core, self.stats
        _, bytes_used, stats.offered, stats.admitted, stats.duplicates = core.counters()
        stats.peak_bytes = bytes_used
        stats.levels = self.cache.stats_rows()
        stats.search_seconds = time.perf_counter() - self._t_search
        if hasattr(core, "transfer_stats"):
            stats.h2d_bytes, stats.d2h_bytes = core.transfer_stats()
        if self._traces is not None:  # the upload of the character matrices and the counters read back belong to the search
            ti = self._traces.info()
            stats.h2d_bytes += ti["h2d_bytes"]
            stats.d2h_bytes += ti["d2h_bytes"]
        if not self.keep_core:
            close = getattr(core, "close", None)
            if close:
                t_close = time.perf_counter()
                close()
                stats.phase_ms["close"] = 1e3 * (time.perf_counter() - t_close)
        return outcome

    keep_core = False
    #: run the cost-level loop inside the library (`ltl_core_run_search`) when the core offers it; False: one
    #: `run_level` call per level from this module (what cores without `run_search` -- oracle, sharded -- always get)
    native_loop = True

    def _run_in_core(self, ops, atom_c: int) -> EnumOutcome:
        """The level loop of `run` as one library call (reference `enumerator.py:234-251`): same segments, same
        bookkeeping, no interpreter between the levels."""
        cfg, cache, core, stats = self.cfg, self.cache, self.core, self.stats
        _check_deadline(cfg)
        if cfg.deadline is not None:
            core.set_option("deadline_ms", max(1, int(1e3 * (cfg.deadline - time.monotonic()))))
        op_cost = [cfg.cost.of(op) for op in range(8)]
        mask = sum(1 << op for op in ops)
        status, op, li, ri, end_cost, rows = core.run_search(op_cost, mask, cache.buckets(), atom_c + 1, self.ceiling,
                                                             cfg.store_last_level)
        cache.absorb_levels(rows)
        if status == S_TIMEOUT:
            raise TimeoutExceeded("learner deadline exceeded")
        if status == S_OOM:
            start = max((rng[1] for rng in cache._buckets.values()), default=0)  # begin_level of the level that ran out
            cache._buckets.setdefault(end_cost, [start, start])
            self.outcome = self._finish(OutOfMemory(stats))
        elif status == S_SOLVED:
            self.outcome = self._finish(Solved(cache.build_candidate(op, li, ri), end_cost, stats))
        else:
            self.outcome = self._finish(CeilingReached(self.spec, self.alphabet, self.ceiling, stats))
        return self.outcome

    def run(self) -> EnumOutcome:
        if self.outcome is not None:
            return self.outcome
        cfg, cache, core, stats = self.cfg, self.cache, self.core, self.stats
        ops = enabled_ops(cfg)
        atom_c = cfg.cost.of(OP_ATOM)
        if self.native_loop and hasattr(core, "run_search"):
            return self._run_in_core(ops, atom_c)
        for c in range(atom_c + 1, self.ceiling):
            _check_deadline(cfg)
            t0 = time.perf_counter()
            cache.begin_level(c)
            if c == self.ceiling - 1 and not cfg.store_last_level and hasattr(core, "set_option"):
                core.set_option("store_results", 0)
            hit = _run_level(core, level_segments(cache, cfg, ops, c), cfg)
            if hit is not None:
                status, op, li, ri = hit
                if status == S_OOM:
                    self.outcome = self._finish(OutOfMemory(stats))
                    return self.outcome
                formula = cache.build_candidate(op, li, ri)
                cache.end_level(c)
                self.outcome = self._finish(Solved(formula, c, stats))
                return self.outcome
            cache.end_level(c)
            cache._rows[-1]["ms"] = round((time.perf_counter() - t0) * 1e3, 3)
        self.outcome = self._finish(CeilingReached(self.spec, self.alphabet, self.ceiling, stats))
        return self.outcome


def enum_learn(spec: Specification, alphabet: Alphabet, cfg: LearnerConfig | None = None, *,
               core_factory: Callable | None = None) -> EnumOutcome:
    """Learn a separating formula, or report OOM / fall back to the overfitting formula (reference
    `enumerator.py:159-251`)."""
    return Enumeration(spec, alphabet, cfg, core_factory=core_factory).run()


# ---------------------------------------------------------------------------------- learn()


@dataclass
class LearnResult:
    """What `learn` returns.  ``status`` is "solved" (``formula`` is a minimal-cost sound formula
    within ``max_cost``), "ceiling" (none exists within ``max_cost``; ``formula`` is the overfitting
    formula, sound but above the cost bound) or "oom" (budget exhausted, no formula)."""

    status: str
    formula: Optional[Formula]
    text: Optional[str]
    cost: Optional[int]
    stats: EnumStats

    def __bool__(self):
        return self.status == "solved"


#: array-pair inputs of at least this many characters are uploaded and checked on the device (`core.DeviceTraces`)
DEVICE_SPEC_MIN_CHARS = 1 << 16


def _is_array_pair(x) -> bool:
    return isinstance(x, tuple) and len(x) == 2 and isinstance(x[0], np.ndarray) and x[0].ndim == 2


def as_specification(P, N, device: int | None = None) -> Specification:
    """``P`` a `Specification` (``N`` None), two iterables of traces, or two ``(chars uint16[k, L], lengths[k])`` array
    pairs; array pairs are uploaded to ``device`` (when given) and checked there (`Specification.from_arrays`)."""
    if isinstance(P, Specification) and N is None:
        return P
    if _is_array_pair(P) and _is_array_pair(N):
        # small specifications are checked faster by numpy than by three kernels and two round trips (config 1: 16 traces)
        if P[0].size + N[0].size < DEVICE_SPEC_MIN_CHARS:
            device = None
        return Specification.from_arrays(P[0], P[1], N[0], N[1], device=device)
    return Specification(P, N)


def learn(P, N=None, alphabet: Alphabet | int | Sequence[str] | None = None, max_cost: int | None = None,
          costs: CostHomomorphism | Sequence[int] | None = None, *, require_nnf: bool = False,
          forbid_until: bool = False, noise: float = 0.0, hash: HashScheme | None = None,
          budget_bytes: int | None = None, deadline_s: float | None = None, device: int = 0,
          overfit_on_ceiling: bool = True, store_last_level: bool = False,
          core_factory: Callable | None = None) -> LearnResult:
    """Learn a minimal LTL formula accepting every trace in ``P`` and rejecting every trace in ``N``.

    ``P`` / ``N``: iterables of traces (each a sequence of int character bitmasks), ``(chars, lengths)`` array
    pairs (``uint16[k, L]`` character matrix + ``k`` lengths: the form for 10^6 traces, checked and packed on the
    device), or ``P`` a `Specification`.  ``alphabet``: an `Alphabet`, a list of proposition names or a proposition
    count (default: as many as the traces use).  ``max_cost``: inclusive cost bound (the reference's
    exclusive ``ceiling`` is ``max_cost + 1``, `enumerator.py:236`).  ``costs``: 8 per-connective
    weights `(atom, !, &, |, X, F, G, U)`, default uniform.
    """
    spec = as_specification(P, N, device if core_factory is None else None)
    if alphabet is None:
        alphabet = Alphabet.default(spec.char_width())
    elif isinstance(alphabet, int):
        alphabet = Alphabet.default(alphabet)
    elif not isinstance(alphabet, Alphabet):
        alphabet = Alphabet(tuple(alphabet))
    if costs is None:
        costs = UNIFORM
    elif not isinstance(costs, CostHomomorphism):
        costs = CostHomomorphism(tuple(costs))
    cfg = LearnerConfig(cost=costs, require_nnf=require_nnf, forbid_until=forbid_until, noise=noise,
                        hash=hash or HashScheme(), ceiling=None if max_cost is None else int(max_cost) + 1,
                        deadline=None if deadline_s is None else time.monotonic() + deadline_s, device=device,
                        store_last_level=store_last_level,
                        **({} if budget_bytes is None else {"budget_bytes": int(budget_bytes)}))
    out = enum_learn(spec, alphabet, cfg, core_factory=core_factory)
    if isinstance(out, Solved):
        return LearnResult("solved", out.formula, print_formula(out.formula, alphabet), out.cost, out.stats)
    if isinstance(out, OutOfMemory):
        return LearnResult("oom", None, None, None, out.stats)
    f = out.formula if overfit_on_ceiling else None
    return LearnResult("ceiling", f, print_formula(f, alphabet) if f is not None else None,
                       out.stats.ceiling if f is not None else None, out.stats)
