"""CPU: the oracle (oracle/ltl_oracle.c) against the golden vectors produced by running the
reference itself (tests/golden/make_golden.py).  This is what pins the oracle."""
import numpy as np
import pytest

from helpers import cfg_from_golden, golden, oracle_factory, records_array, sha, spec_from_golden, unhex
from oracle import cpu_oracle
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200.formula import print_formula

OPS = {"not": 1, "and": 2, "or": 3, "next": 4, "finally": 5, "globally": 6, "until": 7}


def test_kat_mueller():
    for row in golden()["kat"]["mueller"]:
        words = unhex(row["words"])
        core = cpu_oracle.OracleCore(np.full(len(words), 2**64 - 1, dtype=np.uint64), 1, 0, cpu_oracle.V_MUELLER)
        assert core.fingerprint_of(words) == int(row["fp"], 16)


def test_operator_vectors():
    for case in golden()["opvec"]:
        masks = unhex(case["masks"])
        core = cpu_oracle.OracleCore(masks, case["n_pos"], 0, cpu_oracle.V_MUELLER)
        x, y = unhex(case["x"]), unhex(case["y"])
        for name, op in OPS.items():
            got = core.apply_unary(op, x) if op in (1, 4, 5, 6) else core.apply_binary(op, x, y)
            assert (got == unhex(case[name])).all(), name
        assert core.errors(x) == case["errors_x"]


def test_fingerprint_vectors():
    for case in golden()["fpvec"]:
        core = cpu_oracle.OracleCore(unhex(case["masks"]), 1, 0, case["variant"], case["proj_rows"], case["proj_offs"],
                                     case["fkp_bits"], case["mask_k"])
        for cm, fp, fpi in zip(case["cms"], case["fps"], case["fps_int"]):
            assert fp == fpi
            assert core.fingerprint_of(unhex(cm)) == int(fp, 16)


def _replay_transcript(core, tr):
    seeds = [unhex(c) for c in tr["seeds"]]
    k = 0
    n0 = n1 = None
    binaries = 0
    for step in tr["log"]:
        if step[0] == "add":
            assert core.add_entry(seeds[k], 0, k, -1) == step[1]
            k += 1
            continue
        if n0 is None:
            n0 = core.n_entries
        if step[0] == "unary":
            assert list(core.screen_unary(step[1], 0, n0)) == step[2]
            continue
        if n1 is None:
            n1 = core.n_entries
        binaries += 1
        if binaries <= 3:
            tri = step[1] in (2, 3)
            got = core.screen_binary(step[1], 0, n0, 0, n0, tri)
        elif binaries == 4:
            got = core.screen_binary(2, 0, n0, n0, n1, False)
        else:
            got = core.screen_binary(7, n0, n1, 0, n0, False)
        assert list(got) == step[2]


@pytest.mark.parametrize("threads", [1, 4])
def test_transcripts_full(threads):
    for tr in golden()["transcripts"]:
        core = cpu_oracle.OracleCore(unhex(tr["masks"]), tr["n_pos"], 0, cpu_oracle.V_MUELLER, budget_bytes=1 << 24,
                                     threads=threads)
        _replay_transcript(core, tr)
        assert core._counters() == tr["counters"]
        assert sha(core.export_cms()) == tr["cms_sha"]
        assert sha(records_array(core)) == tr["records_sha"]


@pytest.mark.parametrize("case", golden()["learn"], ids=lambda c: c["name"])
def test_learn_cases_with_oracle_core(case):
    if case["stats"]["offered"] > 300000:
        pytest.skip("large case covered by the threaded run below")
    _check_learn(case, threads=1)


@pytest.mark.parametrize("name", ["simple3_k6_s1", "simple3_k6_s3", "noise10"])
def test_learn_large_cases_threaded(name):
    case = next(c for c in golden()["learn"] if c["name"] == name)
    _check_learn(case, threads=8)


def _check_learn(case, threads):
    spec, alphabet = spec_from_golden(case)
    cfg = cfg_from_golden(case["cfg"])
    cores = []
    make = oracle_factory(threads)

    def factory(*a, **kw):
        cores.append(make(*a, **kw))
        cores[-1].close = lambda: None  # keep alive for inspection
        return cores[-1]

    out = L.enum_learn(spec, alphabet, cfg, core_factory=factory)
    assert type(out).__name__ == case["outcome"]
    st = out.stats.as_dict()
    for k, v in case["stats"].items():
        assert st[k] == v, k
    got_levels = [{k: v for k, v in lv.items() if k != "ms"} for lv in out.stats.levels]
    assert got_levels == case["levels"]
    if case["outcome"] == "Solved":
        assert print_formula(out.formula, alphabet) == case["formula"]
        assert out.cost == case["cost"]
    if case["outcome"] == "CeilingReached":
        assert out.ceiling == case["ceiling"]
        assert len(print_formula(out.formula, alphabet)) == case["formula_len"]
    if "core" in case:
        core = cores[-1]
        g = case["core"]
        assert core.n_entries == g["n_entries"]
        assert sha(core.export_cms()) == g["cms_sha"]
        assert sha(records_array(core)) == g["records_sha"]


# ---- NH fingerprint (this build's hash beyond the reference's domain; no reference counterpart)

_M = (1 << 64) - 1


def _mix64(x):
    x ^= x >> 30
    x = x * 0xBF58476D1CE4E5B9 & _M
    x ^= x >> 27
    x = x * 0x94D049BB133111EB & _M
    return x ^ (x >> 31)


def _nh_python(cm):
    """Independent restatement of oracle/ltl_oracle.c fp_nh on Python ints."""
    step, seed0 = 0x9E3779B97F4A7C15, 0x243F6A8885A308D3
    key = [_mix64(((j + 1) * step + seed0) & _M) for j in range(65)]
    s0 = s1 = d0 = d1 = 0
    for k, x in enumerate(int(v) for v in cm):
        p, xl, xh = k & 63, x & 0xFFFFFFFF, x >> 32
        d0 = (d0 + ((xl + (key[p] & 0xFFFFFFFF)) & 0xFFFFFFFF) * ((xh + (key[p] >> 32)) & 0xFFFFFFFF)) & _M
        d1 = (d1 + ((xl + (key[p + 1] & 0xFFFFFFFF)) & 0xFFFFFFFF) * ((xh + (key[p + 1] >> 32)) & 0xFFFFFFFF)) & _M
        if p == 63 or k + 1 == len(cm):
            u = ((k >> 6) + 1) * step & _M
            s0 = (s0 + _mix64(d0 ^ u)) & _M
            s1 = (s1 + _mix64((d1 + u) & _M)) & _M
            d0 = d1 = 0
    return ((_mix64(s0) & ((1 << 62) - 1)) << 64) | _mix64(s1)


def test_nh_fingerprint_known_answers_and_restatement():
    assert _nh_python(np.zeros(1, dtype=np.uint64)) == 0x347E3C3F0D6351A09671A12CA210CF9D
    assert _nh_python(np.arange(100, dtype=np.uint64)) == 0x1922593D4DD0549A2DB84339420886A9
    rng = np.random.default_rng(0)
    for R, W in [(1, 1), (3, 1), (64, 1), (65, 1), (200, 3), (1024, 1), (33, 16)]:
        core = cpu_oracle.OracleCore(np.full(R * W, 2**64 - 1, dtype=np.uint64), 1, 0, cpu_oracle.V_NH, words_per_row=W)
        for _ in range(3):
            cm = rng.integers(0, 1 << 63, size=R * W, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=R * W, dtype=np.uint64)
            assert core.fingerprint_of(cm) == _nh_python(cm)
            # position dependence: swapping two different words changes the value
            sw = cm.copy()
            if R * W > 1 and sw[0] != sw[-1]:
                sw[0], sw[-1] = cm[-1], cm[0]
                assert core.fingerprint_of(sw) != core.fingerprint_of(cm)


def test_scheme_selects_nh_only_beyond_the_reference_domain():
    from paper_2402_12373_b200 import scheme as S

    long_rows = [63] * 64
    assert S.resolve_scheme(S.HashScheme(), long_rows).variant == S.V_MUELLER          # 64 words: the reference's hash
    assert S.resolve_scheme(S.HashScheme(), [63] * 65).variant == S.V_NH               # 65 words: outside its domain
    assert S.resolve_scheme(S.HashScheme(), long_rows, words_per_row=2).variant == S.V_NH
    assert S.resolve_scheme(S.HashScheme("mueller_blocked"), [63] * 65).variant == S.V_MUELLER
    assert S.resolve_scheme(S.HashScheme("nh"), long_rows).variant == S.V_NH
    assert S.resolve_scheme(S.HashScheme("fkp"), [63] * 65).variant == S.V_FKP
    assert S.resolve_scheme(S.HashScheme(), [5] * 8).variant == S.V_GATHER              # precise mode is unaffected


def test_nh32_is_nh_over_row_pairs():
    """V_NH32 (traces of at most 32 positions): NH over virtual words holding two rows each -- the value the device's
    half-width store hashes.  Independent restatement: pack the pairs in numpy, hash with the Python NH above."""
    from paper_2402_12373_b200 import scheme as S

    rng = np.random.default_rng(5)
    for R in (1, 2, 3, 64, 65, 127, 128, 129, 1000, 1025):
        core = cpu_oracle.OracleCore(np.full(R, 0xFFFFFFFF00000000, dtype=np.uint64), 1, 0, cpu_oracle.V_NH32)
        for _ in range(3):
            cm = rng.integers(0, 1 << 32, size=R, dtype=np.uint64) << np.uint64(32)
            padded = np.concatenate([cm, np.zeros(R % 2, dtype=np.uint64)])
            virtual = padded[0::2] | (padded[1::2] >> np.uint64(32))
            assert core.fingerprint_of(cm) == _nh_python(virtual)
    assert S.resolve_scheme(S.HashScheme(), [32] * 65).variant == S.V_NH32
    assert S.resolve_scheme(S.HashScheme(), [33] * 65).variant == S.V_NH
    assert S.resolve_scheme(S.HashScheme(), [32] * 64).variant == S.V_MUELLER      # inside the reference's domain
    assert S.resolve_scheme(S.HashScheme("nh"), [20] * 40).variant == S.V_NH32
    assert S.resolve_scheme(S.HashScheme("mueller_blocked"), [32] * 65).variant == S.V_MUELLER
    with pytest.raises(ValueError):
        cpu_oracle.OracleCore(np.zeros(4, dtype=np.uint64), 1, 0, cpu_oracle.V_NH32, words_per_row=2)
