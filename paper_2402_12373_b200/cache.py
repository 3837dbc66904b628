"""Cost-indexed bookkeeping over the screening core's append-only entry store.

The core (device-resident for the product path) owns matrices, records and the uniqueness set;
this class only tracks which contiguous entry-index range belongs to which formula cost, the
per-level statistics rows, and rebuilds formulae from records.  Contract: reference
`cache.py:101-213` (`try_admit` 124-140, `begin_level`/`end_level` 144-166, `bucket_range`
170-172, `reconstruct`/`build_candidate` 197-213).
"""
from __future__ import annotations

import numpy as np

from .formula import OP_ATOM, UNARY_OPS, Atom, Formula, make_binary, make_unary


class LanguageCache:
    def __init__(self, core):
        self.core = core
        self._buckets: dict[int, list[int]] = {}
        self._frontier = 0
        self._rows: list[dict] = []
        self._mark = (0, 0, 0)

    # -- admission of single matrices (atoms) ------------------------------------------
    def try_admit(self, cm, record, cost: int) -> bool:
        op, lhs, rhs = record
        if cost < self._frontier:
            raise ValueError(f"bucket for cost {cost} is frozen")
        return self._book(self.core.add_entry(np.asarray(cm, dtype=np.uint64), op, lhs, rhs), cost)

    def try_admit_atom(self, traces, prop: int, negated: bool, record, cost: int) -> bool:
        """`try_admit` of a proposition's matrix (or its negation) taken from device-resident packed traces
        (`CudaCore.add_atom`): no matrix crosses the host."""
        op, lhs, rhs = record
        if cost < self._frontier:
            raise ValueError(f"bucket for cost {cost} is frozen")
        return self._book(self.core.add_atom(traces, prop, negated, op, lhs, rhs), cost)

    def _book(self, idx: int, cost: int) -> bool:
        if idx < 0:
            return False
        rng = self._buckets.setdefault(cost, [idx, idx])
        if rng[1] != idx:
            raise AssertionError("non-contiguous admission order")
        rng[1] = idx + 1
        self._frontier = cost
        return True

    # -- level bookkeeping -------------------------------------------------------------
    def begin_level(self, cost: int, counters=None):
        if cost < self._frontier:
            raise ValueError("cost levels must not decrease")
        self._frontier = cost
        n, _, offered, admitted, duplicates = counters or self.core.counters()
        self._buckets.setdefault(cost, [n, n])
        self._mark = (offered, admitted, duplicates)

    def end_level(self, cost: int, counters=None):
        n, bytes_used, offered, admitted, duplicates = counters or self.core.counters()
        self._buckets[cost][1] = n
        o0, a0, d0 = self._mark
        self._rows.append({"cost": cost, "offered": offered - o0, "admitted": admitted - a0,
                           "duplicates": duplicates - d0, "bytes": bytes_used})
        self._frontier = cost + 1

    def absorb_levels(self, rows):
        """Bookkeeping of cost levels that ran inside the core (`CudaCore.run_search`): their buckets and stats rows."""
        for r in rows:
            first, end = r["entries"]
            self._buckets[r["cost"]] = [int(first), int(end)]
            row = {"cost": r["cost"], "offered": r["offered"], "admitted": r["admitted"], "duplicates": r["duplicates"],
                   "bytes": r["bytes"]}
            if r.get("status", 0) == 0:
                row["ms"] = r["ms"]
            self._rows.append(row)
            self._frontier = r["cost"] + 1

    def buckets(self) -> dict:
        return {c: (rng[0], rng[1]) for c, rng in self._buckets.items()}

    def bucket_range(self, cost: int) -> tuple[int, int]:
        got = self._buckets.get(cost)
        return (got[0], got[1]) if got else (0, 0)

    def stats_rows(self) -> list[dict]:
        return list(self._rows)

    def bucket_checksum(self, cost: int) -> int:
        s, e = self.bucket_range(cost)
        if s == e:
            return 0
        return int(np.bitwise_xor.reduce(self.core.export_cms(s, e - s), axis=None))

    # -- reconstruction ----------------------------------------------------------------
    def reconstruct(self, idx: int) -> Formula:
        n = self.core.n_entries
        memo: dict[int, Formula] = {}
        todo = [int(idx)]
        recs: dict[int, tuple] = {}
        if hasattr(self.core, "get_subtree"):  # every record of the formula in one device round trip
            try:
                recs = self.core.get_subtree(int(idx))
            except IndexError:
                recs = {}
        while todo:
            e = todo[-1]
            if e in memo:
                todo.pop()
                continue
            rec = recs.get(e)
            if rec is None:
                rec = recs[e] = tuple(int(v) for v in self.core.get_record(e))
            op, lhs, rhs = rec
            if op == OP_ATOM:
                memo[e] = Atom(lhs)
                todo.pop()
                continue
            kids = (lhs,) if op in UNARY_OPS else (lhs, rhs)
            if any(k < 0 or k >= n for k in kids):
                raise IndexError(f"dangling child reference in entry {e}")
            missing = [k for k in kids if k not in memo]
            if missing:
                todo.extend(missing)
                continue
            memo[e] = make_unary(op, memo[lhs]) if op in UNARY_OPS else make_binary(op, memo[lhs], memo[rhs])
            todo.pop()
        return memo[int(idx)]

    def build_candidate(self, op: int, lhs: int, rhs: int) -> Formula:
        if op in UNARY_OPS:
            return make_unary(op, self.reconstruct(lhs))
        return make_binary(op, self.reconstruct(lhs), self.reconstruct(rhs))
