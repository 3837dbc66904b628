"""Device-resident specification (`include/ltl_core.h: ltl_traces_*`, `core.DeviceTraces`) against the host rules.

What the reference does on the host before a search -- de-duplication and the P/N clash check of `Specification`
(reference `traces.py:64-106`), the census of the overfit cost (`formula.py:230-250`), trace packing
(`bitsem.py:73-88`), the atom fast path (`enumerator.py:182-192`), the admission of the atoms (`218-232`) -- is checked
here on the device path against the host path of this repository (itself pinned to the reference by
tests/test_host_cpu.py) and, for whole searches, against the CPU oracle.
"""
import warnings

import numpy as np
import pytest

from helpers import oracle_factory
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200.packing import TraceContext
from paper_2402_12373_b200.traces import Alphabet, Specification

pytestmark = pytest.mark.gpu


def _random_arrays(rng, n_props, n_pos, n_neg, lo, hi, width=None, junk=True):
    """Distinct random traces as (chars, lengths) pairs; lo == 0 puts one empty trace among the negatives.  Rows that
    repeat an earlier trace are redrawn (with a length from the upper half of the range)."""
    width = width or hi
    R = n_pos + n_neg
    lengths = rng.integers(max(lo, 1), hi + 1, size=R).astype(np.int64)
    if lo == 0 and n_neg:
        lengths[R - 1] = 0
    chars = rng.integers(0, 1 << n_props, size=(R, width)).astype(np.uint16)
    seen = set()
    for r in range(R):
        for _attempt in range(1000):
            key = (int(lengths[r]), chars[r, : lengths[r]].tobytes())
            if key not in seen:
                seen.add(key)
                break
            lengths[r] = rng.integers(max((lo + hi) // 2, 1), hi + 1)
            chars[r] = rng.integers(0, 1 << n_props, size=width)
        else:
            raise AssertionError("could not draw distinct traces: shape too small for that many rows")
    clean = chars * (np.arange(width)[None, :] < lengths[:, None]).astype(np.uint16)
    use = chars if junk else clean  # junk beyond the lengths must be ignored by the device
    return (use[:n_pos].copy(), lengths[:n_pos].copy()), (use[n_pos:].copy(), lengths[n_pos:].copy())


@pytest.mark.parametrize("n_props,n_pos,n_neg,lo,hi,width", [
    (1, 1, 1, 1, 1, 1), (2, 8, 8, 1, 16, 16), (3, 100, 57, 0, 64, 64), (3, 33, 90, 0, 63, 70), (4, 700, 900, 0, 32, 32),
    (2, 40, 40, 60, 200, 200), (5, 300, 10, 1, 130, 1024), (16, 50, 50, 0, 20, 24), (3, 5000, 7000, 3, 40, 40),
])
def test_census_and_packing_match_host(n_props, n_pos, n_neg, lo, hi, width):
    rng = np.random.default_rng(n_pos * 131 + hi)
    P, N = _random_arrays(rng, n_props, n_pos, n_neg, lo, hi, width)
    host = Specification.from_arrays(P[0], P[1], N[0], N[1])
    dev = Specification.from_arrays(P[0], P[1], N[0], N[1], device=0)
    assert dev.device_traces is not None and dev._chars is None  # nothing concatenated on the host yet
    assert (dev.n_pos, dev.n_neg, dev.size) == (host.n_pos, host.n_neg, host.size)
    assert dev.max_len == host.max_len
    assert dev.char_width() == host.char_width()
    assert dev.positive_char_census() == host.positive_char_census()
    assert dev.n_nonempty == host.n_nonempty and dev.n_empty_positive == host.n_empty_positive == 0
    alphabet = Alphabet.default(n_props)
    want = TraceContext.from_spec(host, alphabet)
    dev.device_traces.pack(n_props)
    info = dev.device_traces.info()
    assert info["words"] == want.words
    masks, atoms = dev.device_traces.export()
    assert (masks == want.masks).all()
    assert (atoms == want.atoms).all()
    for p in range(n_props):
        assert info["atom_errors"][p] == L._host_error_count(want.atoms[p], host.n_pos)
        assert info["neg_atom_errors"][p] == L._host_error_count(~want.atoms[p] & want.masks, host.n_pos)
    # the lazily concatenated host view is the canonical (zero-padded) matrix of the host path
    assert (dev.lengths == host.lengths).all()
    assert (dev.chars[:, : host.chars.shape[1]] == host.chars).all() and not dev.chars[:, host.chars.shape[1]:].any()
    assert info["h2d_bytes"] >= (n_pos + n_neg) * min(width, max(host.max_len, 0)) * 2  # columns no trace reaches stay home
    dev.release_device()
    assert dev.device_traces is None


def test_duplicates_and_clashes_follow_the_host_rules():
    rng = np.random.default_rng(7)
    P, N = _random_arrays(rng, 3, 300, 300, 1, 20, 20)
    pc, pl = np.concatenate([P[0], P[0][5:8]]), np.concatenate([P[1], P[1][5:8]])  # three duplicate positives
    nc, nl = np.concatenate([N[0][:1], N[0]]), np.concatenate([N[1][:1], N[1]])    # one duplicate negative
    with warnings.catch_warnings(record=True) as w_host:
        warnings.simplefilter("always")
        host = Specification.from_arrays(pc, pl, nc, nl)
    with warnings.catch_warnings(record=True) as w_dev:
        warnings.simplefilter("always")
        dev = Specification.from_arrays(pc, pl, nc, nl, device=0)
    assert sorted(str(w.message) for w in w_dev) == sorted(str(w.message) for w in w_host) and len(w_host) == 2
    assert (dev.n_pos, dev.n_neg) == (host.n_pos, host.n_neg) == (300, 300)
    assert (dev.chars == host.chars).all() and (dev.lengths == host.lengths).all()
    assert dev.device_traces is not None and dev.device_traces.info()["rows"] == 600
    # junk beyond the length does not make traces different
    pc2 = pc.copy()
    short = int(np.argmin(pl[:300]))
    if pl[short] < 20:
        pc2[short, pl[short]:] ^= 1
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            again = Specification.from_arrays(pc2, pl, nc, nl, device=0)
        assert again.n_pos == 300
    # a trace on both sides is refused, with the host's message
    nc3, nl3 = np.concatenate([N[0], P[0][17:18]]), np.concatenate([N[1], P[1][17:18]])
    with pytest.raises(ValueError) as e_host:
        Specification.from_arrays(P[0], P[1], nc3, nl3)
    with pytest.raises(ValueError) as e_dev:
        Specification.from_arrays(P[0], P[1], nc3, nl3, device=0)
    assert str(e_dev.value) == str(e_host.value) and "both sides" in str(e_dev.value)


def _summary(res):
    rows = [{k: v for k, v in r.items() if k != "ms"} for r in res.stats.levels]
    return (res.status, res.text, res.cost, res.stats.offered, res.stats.admitted, res.stats.duplicates,
            res.stats.atom_fast_path, res.stats.precise, res.stats.ceiling, rows)


LEARN_CASES = [
    dict(seed=1, n_props=2, n_pos=40, n_neg=50, lo=1, hi=12, kw=dict(max_cost=6)),
    dict(seed=2, n_props=3, n_pos=200, n_neg=180, lo=0, hi=30, kw=dict(max_cost=5)),                     # NH32 store
    dict(seed=3, n_props=2, n_pos=60, n_neg=60, lo=40, hi=150, kw=dict(max_cost=5)),                     # 3 words per row
    dict(seed=4, n_props=2, n_pos=90, n_neg=70, lo=1, hi=40, kw=dict(max_cost=6, noise=0.15)),
    dict(seed=5, n_props=2, n_pos=80, n_neg=80, lo=1, hi=25, kw=dict(max_cost=6, require_nnf=True)),      # negated atoms
    dict(seed=6, n_props=2, n_pos=50, n_neg=50, lo=1, hi=25, kw=dict(max_cost=5, forbid_until=True)),
    dict(seed=7, n_props=2, n_pos=5, n_neg=4, lo=1, hi=6, kw=dict(max_cost=7)),                           # gather (precise)
    dict(seed=8, n_props=2, n_pos=64, n_neg=64, lo=1, hi=50, kw=dict(max_cost=5, budget_bytes=2 * (128 * 8 + 16) + 1)),
    dict(seed=9, n_props=2, n_pos=64, n_neg=64, lo=1, hi=50, kw=dict(max_cost=5, budget_bytes=40 * (128 * 8 + 16) + 1)),
    dict(seed=10, n_props=3, n_pos=120, n_neg=100, lo=2, hi=20, kw=dict(max_cost=8), planted="F(p0 & X p1)"),
    dict(seed=11, n_props=3, n_pos=120, n_neg=100, lo=2, hi=20, kw=dict(max_cost=8), planted="p2"),       # atom fast path
    dict(seed=12, n_props=3, n_pos=120, n_neg=100, lo=2, hi=20, kw=dict(max_cost=8, require_nnf=True), planted="!p1"),
    dict(seed=13, n_props=2, n_pos=150, n_neg=150, lo=2, hi=20, kw=dict(max_cost=8, noise=0.2), planted="p0 U p1"),
]


@pytest.mark.parametrize("case", LEARN_CASES, ids=[str(c["seed"]) for c in LEARN_CASES])
def test_learn_from_arrays_matches_host_path_and_oracle(case, monkeypatch):
    """`learn((chars, lengths), (chars, lengths), ...)`: the specification is uploaded, checked, packed and searched on
    the device -- same outcome, counters and per-level rows as the host-packed search and as the CPU oracle."""
    from paper_2402_12373_b200 import workloads as Wl

    if "planted" in case:
        spec, alphabet, _ = Wl.planted_spec(case["n_props"], case["n_pos"], case["n_neg"], case["lo"], case["hi"],
                                            case["planted"], case["seed"])
        P = (spec.chars[: spec.n_pos].copy(), spec.lengths[: spec.n_pos].copy())
        N = (spec.chars[spec.n_pos:].copy(), spec.lengths[spec.n_pos:].copy())
    else:
        P, N = _random_arrays(np.random.default_rng(case["seed"]), case["n_props"], case["n_pos"], case["n_neg"],
                              case["lo"], case["hi"])
        alphabet = Alphabet.default(case["n_props"])
    monkeypatch.setattr(L, "DEVICE_SPEC_MIN_CHARS", 0)  # these small inputs must take the device-resident path
    host_spec = Specification.from_arrays(P[0], P[1], N[0], N[1])
    want = _summary(L.learn(host_spec, None, alphabet, core_factory=oracle_factory(2), **case["kw"]))
    host = L.learn(host_spec, None, alphabet, **case["kw"])
    got = L.learn(P, N, alphabet, **case["kw"])
    assert _summary(host) == want
    assert _summary(got) == want
    assert got.stats.h2d_bytes >= host_spec.size * host_spec.max_len * 2  # the character matrix went to the device
    if got.status == "solved":
        assert Wl.error_count(got.formula, host_spec, alphabet) <= int(case["kw"].get("noise", 0.0) * host_spec.size + 1e-9)


def test_resident_specification_serves_several_searches():
    P, N = _random_arrays(np.random.default_rng(21), 2, 70, 70, 1, 30)
    spec = Specification.from_arrays(P[0], P[1], N[0], N[1], device=0)
    a = L.learn(spec, None, 2, max_cost=5)
    b = L.learn(spec, None, 3, max_cost=5)              # wider alphabet: packed again with three propositions
    c = L.learn(spec, None, 2, max_cost=5, require_nnf=True)
    host = Specification.from_arrays(P[0], P[1], N[0], N[1])
    assert _summary(a) == _summary(L.learn(host, None, 2, max_cost=5))
    assert _summary(b) == _summary(L.learn(host, None, 3, max_cost=5))
    assert _summary(c) == _summary(L.learn(host, None, 2, max_cost=5, require_nnf=True))
