"""GPU: the BASELINE configurations at FULL size and bench depth, against the committed oracle fixture
tests/golden/full_levels.json (made by tests/golden/make_full_levels.py with the CPU oracle port): status, formula
text, cost, counters, and per cost level {offered, admitted, duplicates, bytes, entry range, SHA-256 of the
(op, lhs, rhs) records} -- records determine the matrices inductively, so equal hashes are equal sets of unique CS
in equal order.  One core, and 2 / 4 row shards (virtual ranks on threads, each a real CudaCore on cuda:0).
Plus size-independent properties on config 4 (idempotent re-screening, distinct fingerprints, membership)."""
import functools
import json
import os
import threading

import numpy as np
import pytest

from helpers import ROOT, search_with_record_hashes
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200 import workloads as Wl
from paper_2402_12373_b200.core import make_core
from paper_2402_12373_b200.scheme import HashScheme

pytestmark = pytest.mark.gpu

with open(os.path.join(ROOT, "tests", "golden", "full_levels.json")) as _fh:
    FIXTURE = json.load(_fh)

KEYS = ("status", "formula", "cost", "offered", "admitted", "duplicates", "atoms_sha256", "levels")


@functools.lru_cache(maxsize=2)
def _workload(config: str, random: bool):
    wl = dict(Wl.CONFIGS[config])
    if random:
        return Wl.random_spec(wl["n_props"], wl["n_pos"], wl["n_neg"], wl["min_len"], wl["max_len"], wl["seed"])
    spec, alphabet, _planted, _ = Wl.make_config(config)
    return spec, alphabet


def _assert_same(got: dict, want: dict):
    for k in ("status", "formula", "cost", "offered", "admitted", "duplicates", "atoms_sha256"):
        assert got[k] == want[k], (k, got[k], want[k])
    assert len(got["levels"]) == len(want["levels"])
    for g, w in zip(got["levels"], want["levels"]):
        assert g == w, (g, w)


@pytest.mark.parametrize("case", sorted(FIXTURE))
def test_full_size_levels_and_record_hashes(case):
    want = FIXTURE[case]
    spec, alphabet = _workload(want["config"], want["random"])
    got = search_with_record_hashes(spec, alphabet, max_cost=want["max_cost"], budget_bytes=want["budget_bytes"],
                                    hash=HashScheme(want["hash"]))
    _assert_same(got, want)


SHARDED_CASES = [c for c in ("c2_planted", "c3_long", "c4_many", "c5_deep", "c5_deep_budget", "c5_random_budget")
                 if c in FIXTURE]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", SHARDED_CASES)
def test_full_size_row_sharded(case, world):
    """The same searches over G row shards (every shard holds R / G rows of every matrix; per-candidate partial sums
    added through the exchange callback; fused NOT in phase B on every shard): every rank reproduces the fixture."""
    from paper_2402_12373_b200.sharded import ThreadComm, row_sharded_core_factory

    want = FIXTURE[case]
    spec, alphabet = _workload(want["config"], want["random"])
    comms = ThreadComm.group(world)
    got, errs = [None] * world, []

    def work(r):
        try:
            got[r] = search_with_record_hashes(spec, alphabet, max_cost=want["max_cost"],
                                               budget_bytes=want["budget_bytes"], hash=HashScheme(want["hash"]),
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
        _assert_same(res, want)


def test_bench_bound_gives_the_fixture_result():
    """bench.py runs config 2 with max_cost 12 (the fixture stops at the solving cost 11 so that the oracle never
    stores the last level): same formula, cost and counters."""
    want = FIXTURE["c2_planted"]
    spec, alphabet = _workload("c2_planted", False)
    res = L.learn(spec, None, alphabet, max_cost=Wl.CONFIGS["c2_planted"]["max_cost"], budget_bytes=150 << 30)
    assert (res.status, res.text, res.cost) == (want["status"], want["formula"], want["cost"])
    assert (res.stats.offered, res.stats.admitted, res.stats.duplicates) == (want["offered"], want["admitted"],
                                                                           want["duplicates"])
    assert Wl.error_count(res.formula, spec, alphabet) == 0


def test_hash_schemes_agree_at_full_size():
    """NH (the product default beyond the reference's domain) and blocked MuellerHash produce the same records level
    by level on config 2 in the ORACLE fixtures: no fingerprint collision changed the search."""
    a, b = FIXTURE.get("c2_planted"), FIXTURE.get("c2_planted_mueller_blocked")
    if a is None or b is None:
        pytest.skip("fixture lacks one of the two hash runs")
    _assert_same(a, b)


def test_config4_full_size_row_split_properties():
    """2^20 + 2^20 traces of length 32: every candidate streams MBs, evaluation is split over rows.  Properties
    that need no oracle: idempotent re-screening, pairwise distinct fingerprints, membership."""
    spec, alphabet = _workload("c4_many", False)
    assert spec.size == 1 << 21
    cores = []

    def factory(*a, **kw):
        cores.append(make_core(*a, **kw))
        cores[-1]._real_close, cores[-1].close = cores[-1].close, lambda: None
        return cores[-1]

    got = L.learn(spec, None, alphabet, max_cost=3, core_factory=factory, budget_bytes=64 << 30,
                  overfit_on_ceiling=False, store_last_level=True)
    assert got.status == "ceiling"
    core = cores[-1]
    n = core.n_entries
    before = core.counters()
    st = core.screen_unary(4, 0, 4)  # X over the four atoms again: all duplicates now
    after = core.counters()
    assert st[0] == 0 and after[3] == before[3] and after[4] == before[4] + 4
    hi, lo = core.entry_fingerprints(0, n)
    assert len({(int(a), int(b)) for a, b in zip(hi, lo)}) == n
    a = core.get_cm(0)
    assert core.contains(a) and core.contains((a << np.uint64(1)))  # X p0 was admitted at cost 2
    core._real_close()
    planted = L.learn(spec, None, alphabet, max_cost=Wl.CONFIGS["c4_many"]["max_cost"], budget_bytes=4 << 40)
    assert planted.status == "solved" and Wl.error_count(planted.formula, spec, alphabet) == 0


def test_config2_solves_behind_a_closed_gate(monkeypatch):
    """BASELINE config 2 ends among the AND candidates of cost level 11, in front of the first piece that reads a matrix
    of level 10: the fused phase B of level 10 finds its store gate closed ("gated store") and only screens
    NOT(entry).  Same outcome as a core that always stores (`gate_store=0`) -- the fixture test above holds both to the
    oracle -- and matrices of the level left pending read back identical afterwards."""
    from helpers import LearnerConfig

    spec, alphabet = _workload("c2_planted", False)
    want = FIXTURE["c2_planted"]
    runs = {}
    for gate in (1, 0):
        monkeypatch.setenv("LTL_CORE_OPTIONS", f"gate_store={gate}")
        cfg = LearnerConfig(ceiling=want["max_cost"] + 1, budget_bytes=int(want["budget_bytes"]), hash=HashScheme(want["hash"]))
        en = L.Enumeration(spec, alphabet, cfg)
        en.keep_core = True
        out = en.run()
        s, e = en.cache._buckets[10]
        picks = [s, s + 1, (s + e) // 2, e - 1]  # entries of cost level 10: written only if the gate was open
        runs[gate] = (type(out).__name__, out.cost, out.stats.offered, out.stats.admitted, out.stats.duplicates,
                      en.core.info()["gated_skips"], (int(s), int(e)), [en.core.get_cm(i).copy() for i in picks])
        en.core.close()
    assert runs[1][:5] == runs[0][:5] == ("Solved", want["cost"], want["offered"], want["admitted"], want["duplicates"])
    assert runs[1][5] == 1 and runs[0][5] == 0
    assert runs[1][6] == runs[0][6]
    for a, b in zip(runs[1][7], runs[0][7]):
        assert (a == b).all()
