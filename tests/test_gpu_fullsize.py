"""GPU: the BASELINE configurations at FULL size.  Config 2 (the bench workload) is compared level by level
with a committed fixture produced by the CPU oracle (tests/golden/c2_levels.json, 143 s of CPU); configs 3-5
are compared with the oracle on the levels it finishes in seconds, plus size-independent properties
(soundness of the learned formula on every trace, idempotent re-screening, fingerprint/set consistency)."""
import json
import os

import numpy as np
import pytest

from helpers import ROOT, oracle_factory
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200 import workloads as Wl
from paper_2402_12373_b200.core import make_core
from paper_2402_12373_b200.learner import Segment

pytestmark = pytest.mark.gpu


def _levels(res):
    return [{k: v for k, v in lv.items() if k != "ms"} for lv in res.stats.levels]


def test_config2_full_size_matches_oracle_fixture():
    with open(os.path.join(ROOT, "tests", "golden", "c2_levels.json")) as fh:
        want = json.load(fh)
    spec, alphabet, planted, cfg = Wl.make_config("c2_planted")
    res = L.learn(spec, None, alphabet, max_cost=cfg["max_cost"], budget_bytes=150 << 30)
    assert (res.status, res.text, res.cost) == (want["status"], want["formula"], want["cost"])
    assert (res.stats.offered, res.stats.admitted, res.stats.duplicates) == (want["offered"], want["admitted"],
                                                                           want["duplicates"])
    assert _levels(res) == want["levels"]
    assert Wl.error_count(res.formula, spec, alphabet) == 0


@pytest.mark.parametrize("name,max_cost", [("c3_long", 7), ("c5_deep", 5)])
def test_config3_and_5_full_size_match_oracle(name, max_cost):
    spec, alphabet, planted, cfg = Wl.make_config(name)
    want = L.learn(spec, None, alphabet, max_cost=max_cost, core_factory=oracle_factory(16), budget_bytes=64 << 30,
                   overfit_on_ceiling=False)
    got = L.learn(spec, None, alphabet, max_cost=max_cost, budget_bytes=64 << 30, overfit_on_ceiling=False)
    assert (got.status, got.text, got.cost) == (want.status, want.text, want.cost)
    assert _levels(got) == _levels(want)
    if got.formula is not None:
        assert Wl.error_count(got.formula, spec, alphabet) == 0


def test_config3_full_size_solves_planted_formula():
    spec, alphabet, planted, cfg = Wl.make_config("c3_long")
    res = L.learn(spec, None, alphabet, max_cost=cfg["max_cost"], budget_bytes=150 << 30)
    assert res.status == "solved" and res.cost <= 8
    assert Wl.error_count(res.formula, spec, alphabet) == 0


def test_config4_full_size_row_split_properties():
    """2^20 + 2^20 traces of length 32 (16 MiB per matrix): every candidate streams MBs, evaluation is split
    over rows.  Parity with the oracle on cost levels 2..3; then properties at cost 4."""
    spec, alphabet, planted, cfg = Wl.make_config("c4_many")
    assert spec.size == 1 << 21
    want = L.learn(spec, None, alphabet, max_cost=3, core_factory=oracle_factory(16), budget_bytes=64 << 30,
                   overfit_on_ceiling=False)
    cores = []

    def factory(*a, **kw):
        cores.append(make_core(*a, **kw))
        cores[-1]._real_close, cores[-1].close = cores[-1].close, lambda: None
        return cores[-1]

    got = L.learn(spec, None, alphabet, max_cost=3, core_factory=factory, budget_bytes=64 << 30,
                  overfit_on_ceiling=False, store_last_level=True)
    assert (got.status, got.text) == (want.status, want.text)
    assert _levels(got) == _levels(want)
    core = cores[-1]
    n = core.n_entries
    # idempotence: screening the same unary candidates again admits nothing
    before = core.counters()
    st = core.screen_unary(4, 0, 4)
    after = core.counters()
    assert st[0] == 0 and after[3] == before[3] and after[4] == before[4] + 4
    # fingerprints of stored entries are pairwise distinct (they were admitted as unique)
    hi, lo = core.entry_fingerprints(0, n)
    assert len({(int(a), int(b)) for a, b in zip(hi, lo)}) == n
    # X distributes over &:  X(a & b) == Xa & Xb on every one of the 2^21 rows
    a, b = core.get_cm(0), core.get_cm(1)
    assert core.contains(a) and core.contains((a << np.uint64(1)))  # X p0 was admitted at cost 2
    core._real_close()
    # the logical budget counts admissions of the last level too (reference rule); only levels that serve as
    # operands are ever written, so 4 TB logical fits one GPU here
    planted_res = L.learn(spec, None, alphabet, max_cost=cfg["max_cost"], budget_bytes=4 << 40)
    assert planted_res.status == "solved" and Wl.error_count(planted_res.formula, spec, alphabet) == 0


@pytest.mark.parametrize("world", [2, 4])
def test_config2_full_size_row_sharded(world):
    """The bench workload over G row shards (virtual ranks on threads, each a real CudaCore holding 1024 / G rows of
    every matrix on cuda:0; per-candidate partial sums added through the exchange callback; fused NOT in phase B on
    every shard): level by level the fixture of the single-core run."""
    import threading

    from paper_2402_12373_b200.sharded import ThreadComm, row_sharded_core_factory

    with open(os.path.join(ROOT, "tests", "golden", "c2_levels.json")) as fh:
        want = json.load(fh)
    spec, alphabet, planted, cfg = Wl.make_config("c2_planted")
    comms = ThreadComm.group(world)
    got, errs = [None] * world, []

    def work(r):
        try:
            got[r] = L.learn(spec, None, alphabet, max_cost=cfg["max_cost"], budget_bytes=150 << 30,
                             core_factory=row_sharded_core_factory(comms[r]))
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            comms[r]._s.barrier.abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for res in got:
        assert (res.status, res.text, res.cost) == (want["status"], want["formula"], want["cost"])
        assert (res.stats.offered, res.stats.admitted, res.stats.duplicates) == (want["offered"], want["admitted"],
                                                                               want["duplicates"])
        assert _levels(res) == want["levels"]
