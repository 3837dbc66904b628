"""CPU: tests/golden/full_levels.json is what the oracle produces (the cases it finishes in seconds are regenerated
and compared), its two hash runs of config 2 agree, and the record hash is sensitive to order."""
import json
import os

import numpy as np
import pytest

from helpers import ROOT, oracle_factory, records_sha, search_with_record_hashes
from paper_2402_12373_b200 import workloads as Wl
from paper_2402_12373_b200.scheme import HashScheme

with open(os.path.join(ROOT, "tests", "golden", "full_levels.json")) as _fh:
    FIXTURE = json.load(_fh)

QUICK = ["c1_tiny", "c5_deep", "c5_deep_budget", "c5_random_budget", "c3_random"]


def test_fixture_covers_every_baseline_config():
    assert {"c1_tiny", "c2_planted", "c3_long", "c4_many", "c5_deep"} <= set(FIXTURE)
    for name, case in FIXTURE.items():
        assert case["levels"], name
        for lv in case["levels"]:
            assert len(lv["records_sha256"]) == 64 and lv["entries"][0] <= lv["entries"][1]


@pytest.mark.parametrize("case", QUICK)
def test_oracle_reproduces_fixture(case):
    want = FIXTURE[case]
    wl = dict(Wl.CONFIGS[want["config"]])
    if want["random"]:
        spec, alphabet = Wl.random_spec(wl["n_props"], wl["n_pos"], wl["n_neg"], wl["min_len"], wl["max_len"], wl["seed"])
    else:
        spec, alphabet, _f, _ = Wl.make_config(want["config"])
    got = search_with_record_hashes(spec, alphabet, max_cost=want["max_cost"], budget_bytes=want["budget_bytes"],
                                    core_factory=oracle_factory(4), hash=HashScheme(want["hash"]))
    for k in ("status", "formula", "cost", "offered", "admitted", "duplicates", "atoms_sha256", "levels"):
        assert got[k] == want[k], k


def test_hash_schemes_agree_on_config2():
    a, b = FIXTURE["c2_planted"], FIXTURE["c2_planted_mueller_blocked"]
    assert a["hash"] == "mueller" and b["hash"] == "mueller_blocked"
    for k in ("status", "formula", "cost", "offered", "admitted", "duplicates", "levels"):
        assert a[k] == b[k], k


def test_record_hash_sees_order():
    class Fake:
        def __init__(self, recs):
            self.recs = np.array(recs)

        def export_records(self, first, count):
            r = self.recs[first:first + count]
            return r[:, 0], r[:, 1], r[:, 2]

    a = Fake([(2, 0, 1), (3, 0, 1), (7, 1, 0)])
    b = Fake([(3, 0, 1), (2, 0, 1), (7, 1, 0)])
    assert records_sha(a, 0, 3) != records_sha(b, 0, 3)
    assert records_sha(a, 2, 1) == records_sha(b, 2, 1)
