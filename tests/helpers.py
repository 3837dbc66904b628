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
