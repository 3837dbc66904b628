"""Shared test helpers: golden loader, oracle adapters, seeded spec generators."""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import cpu_oracle  # noqa: E402  (tests are allowed to use the oracle)
from paper_2402_12373_b200 import errors as E  # noqa: E402
from paper_2402_12373_b200.formula import CostHomomorphism  # noqa: E402
from paper_2402_12373_b200.learner import LearnerConfig  # noqa: E402
from paper_2402_12373_b200.scheme import HashScheme  # noqa: E402
from paper_2402_12373_b200.traces import Alphabet, Specification  # noqa: E402

_GOLDEN = None


def golden() -> dict:
    global _GOLDEN
    if _GOLDEN is None:
        with open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")) as fh:
            _GOLDEN = json.load(fh)
    return _GOLDEN


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def unhex(xs) -> np.ndarray:
    return np.array([int(x, 16) for x in xs], dtype=np.uint64)


class OracleAdapter(cpu_oracle.OracleCore):
    """CPU oracle behind the product's core-factory signature (exceptions translated)."""

    def add_entry(self, cm, op, lhs, rhs):
        try:
            return super().add_entry(cm, op, lhs, rhs)
        except cpu_oracle.CoreOOM:
            raise E.CoreOOM from None

    def counters(self):
        return self._counters()


def oracle_factory(threads: int = 1):
    def make(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes, *,
             words_per_row=1, device=None):
        return OracleAdapter(masks, n_pos, err_max, variant, proj_rows, proj_offs, fkp_bits, mask_k, budget_bytes,
                             words_per_row=words_per_row, threads=threads)

    return make


def cfg_from_golden(kw: dict) -> LearnerConfig:
    kw = dict(kw)
    if "hash" in kw:
        kw["hash"] = HashScheme(**kw["hash"])
    if "cost" in kw:
        kw["cost"] = CostHomomorphism(tuple(kw["cost"]))
    kw.setdefault("store_last_level", True)  # the fixtures hash every stored matrix
    return LearnerConfig(**kw)


def spec_from_golden(case: dict):
    return Specification(case["pos"], case["neg"]), Alphabet.default(case["n_props"])


def records_array(core) -> np.ndarray:
    n = core.n_entries
    if hasattr(core, "export_records"):
        op, lhs, rhs = core.export_records(0, n)
        return np.stack([op.astype(np.int64), lhs.astype(np.int64), rhs.astype(np.int64)], axis=1).reshape(-1, 3)
    return np.array([core.get_record(i) for i in range(n)], dtype=np.int64).reshape(-1, 3)


def random_spec(rng, n_props, n_pos, n_neg, lo, hi):
    """Distinct uniformly random traces with lengths in [lo, hi] (positives never empty)."""
    seen, out = set(), []
    while len(out) < n_pos + n_neg:
        length = int(rng.integers(max(lo, 1) if len(out) < n_pos else lo, hi + 1))
        tr = tuple(int(c) for c in rng.integers(0, 1 << n_props, size=length))
        if tr not in seen:
            seen.add(tr)
            out.append(tr)
    return Specification(out[:n_pos], out[n_pos:]), Alphabet.default(n_props)


def records_sha(core, first: int, count: int) -> str:
    """SHA-256 of the (op int8, lhs int32, rhs int32) record arrays of entries [first, first + count): records
    determine the characteristic matrices inductively, so equal hashes level by level mean the same set of
    unique CS in the same order."""
    if count <= 0:
        return hashlib.sha256(b"").hexdigest()
    if hasattr(core, "export_records"):
        op, lhs, rhs = core.export_records(first, count)
    else:
        recs = np.array([core.get_record(first + k) for k in range(count)], dtype=np.int64).reshape(-1, 3)
        op, lhs, rhs = recs[:, 0], recs[:, 1], recs[:, 2]
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(op, dtype=np.int8).tobytes())
    h.update(np.ascontiguousarray(lhs, dtype="<i4").tobytes())
    h.update(np.ascontiguousarray(rhs, dtype="<i4").tobytes())
    return h.hexdigest()


def search_with_record_hashes(spec, alphabet, *, max_cost, budget_bytes, core_factory=None, hash=None, device=0):
    """One search through `learner.Enumeration`; returns the outcome as a JSON-able dict with, per cost level, the
    counters and the SHA-256 of the level's records (fixtures: tests/golden/full_levels.json)."""
    from paper_2402_12373_b200.formula import print_formula
    from paper_2402_12373_b200.learner import Enumeration, OutOfMemory, Solved

    cfg = LearnerConfig(ceiling=max_cost + 1, budget_bytes=int(budget_bytes), hash=hash or HashScheme(), device=device)
    en = Enumeration(spec, alphabet, cfg, core_factory=core_factory)
    en.keep_core = True
    out = en.run()
    status = "solved" if isinstance(out, Solved) else "oom" if isinstance(out, OutOfMemory) else "ceiling"
    res = {"status": status, "formula": print_formula(out.formula, alphabet) if status == "solved" else None,
           "cost": out.cost if status == "solved" else None, "offered": out.stats.offered,
           "admitted": out.stats.admitted, "duplicates": out.stats.duplicates, "levels": []}
    core, cache = en.core, en.cache
    if core is not None:
        n = core.counters()[0]
        s, e = cache.bucket_range(1)
        res["atoms_sha256"] = records_sha(core, s, e - s)
        rows = {r["cost"]: r for r in out.stats.levels}
        costs = sorted(c for c in cache._buckets if c > 1)
        for c in costs:
            s, e = cache._buckets[c]
            e = max(e, s)
            if c not in rows:  # the level a search ended in by OOM has no stats row; its bucket ends at n_entries
                e = n
            row = {k: v for k, v in rows.get(c, {"cost": c}).items() if k != "ms"}
            row["entries"] = [int(s), int(e)]
            row["records_sha256"] = records_sha(core, s, e - s)
            res["levels"].append(row)
        close = getattr(core, "close", None)
        if close:
            close()
    return res
