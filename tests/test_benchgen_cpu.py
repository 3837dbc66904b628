"""Benchmark generators and experiments (`paper_2402_12373_b200/benchgen.py`) against values recorded from the
reference's own `benchgen.py` (tests/golden/make_benchgen_golden.py).  CPU: generators bit for bit; experiments with
the CPU oracle as the screening core on a subset of the recorded rows (the GPU test runs all of them)."""
import json
import os
import warnings

import numpy as np
import pytest

from helpers import oracle_factory
from paper_2402_12373_b200 import benchgen as B
from paper_2402_12373_b200.formula import parse_formula, print_formula
from paper_2402_12373_b200.learner import LearnerConfig
from paper_2402_12373_b200.scheme import HashScheme
from paper_2402_12373_b200.traces import Alphabet, Specification

with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "benchgen_golden.json")) as fh:
    GOLD = json.load(fh)


def as_lists(spec):
    return [list(t) for t in spec.pos], [list(t) for t in spec.neg]


@pytest.mark.parametrize("case", GOLD["simple"], ids=lambda c: f"p{c['n_props']}k{c['k']}s{c['seed']}")
def test_gen_simple_matches_reference(case):
    s = B.gen_simple(Alphabet.default(case["n_props"]), case["k"], case["lo"], case["hi"], case["seed"])
    assert as_lists(s) == (case["pos"], case["neg"])


@pytest.mark.parametrize("case", GOLD["guided"], ids=lambda c: f"{c['formula']}-s{c['seed']}")
def test_gen_guided_matches_reference(case):
    al = Alphabet.default(case["n_props"])
    f = parse_formula(case["formula"], al)
    s = B.gen_guided(al, f, case["k"], case["lo"], case["hi"], case["seed"])
    assert as_lists(s) == (case["pos"], case["neg"])
    assert all(B.trace_cs(f, t) >> (len(t) - 1) & 1 for t in s.pos) and not any(B.trace_cs(f, t) >> (len(t) - 1) & 1 for t in s.neg if t)


@pytest.mark.parametrize("case", GOLD["hamming"], ids=lambda c: f"p{c['n_props']}l{c['l']}d{c['delta']}")
def test_gen_hamming_matches_reference(case):
    s = B.gen_hamming(Alphabet.default(case["n_props"]), case["l"], case["delta"], case["seed"])
    assert as_lists(s) == (case["pos"], case["neg"])


def test_generators_beyond_the_reference_limits_and_errors():
    al = Alphabet.default(2)
    f = parse_formula("p0 U (p1 & X X p0)", al)
    s = B.gen_guided(al, f, 5, 150, 200, 1)  # the reference's evaluator stops at 63 positions
    assert s.n_pos == 5 and s.n_neg == 5 and 150 <= min(len(t) for t in s.pos + s.neg) and s.max_len <= 200
    from paper_2402_12373_b200 import workloads as Wl

    assert Wl.error_count(f, s, al) == 0  # the packed multi-word evaluator agrees with trace_cs
    with pytest.raises(B.GenerationError):
        B.gen_simple(al, 50, 1, 2, 0)  # only 20 traces exist
    with pytest.raises(B.GenerationError):
        B.gen_guided(al, parse_formula("p0 & !p0", al), 1, 3, 5, 0, budget_per_trace=300)
    with pytest.raises(B.GenerationError):
        B.gen_samplebench(9, 1, True, 0)
    with pytest.raises(ValueError):
        B.gen_hamming(al, 4, 0, 5)  # the ball of radius 0 is the positive trace itself (the reference raises too)


def test_trace_cs_agrees_with_the_packed_evaluator():
    from paper_2402_12373_b200 import workloads as Wl
    from paper_2402_12373_b200.packing import TraceContext

    rng = np.random.default_rng(3)
    al = Alphabet.default(3)
    traces = [tuple(int(c) for c in rng.integers(0, 8, size=int(n))) for n in rng.integers(1, 140, size=40)]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = Specification(traces[:20], traces[20:])
    ctx = TraceContext.from_spec(spec, al)
    for text in ["p0 U (p1 & X p2)", "G (p0 | X !p1)", "F G p2", "X X X p0", "!(p0 U p1) | F (p1 & G p0)"]:
        f = parse_formula(text, al)
        cm = Wl.eval_formula(f, ctx)
        for r, tr in enumerate(spec.traces):
            want = 0
            for w in range(cm.shape[1]):
                want = (want << 64) | int(cm[r, w])
            want >>= 64 * cm.shape[1] - len(tr)
            assert B.trace_cs(f, tr) == want, (text, r)


def check_samplebench(case, core_factory):
    sb = B.gen_samplebench(case["i"], case["k"], case["conservative"], case["seed"], core_factory=core_factory)
    a2 = Alphabet.default(2)
    assert print_formula(sb.seed_formula, a2) == case["seed_formula"] and sb.seed_cost == case["seed_cost"]
    assert as_lists(sb.seed_spec) == (case["seed_spec"]["pos"], case["seed_spec"]["neg"])
    assert as_lists(sb.spec) == (case["pos"], case["neg"])


@pytest.mark.parametrize("case", [c for c in GOLD["samplebench"] if c["i"] < 8], ids=lambda c: f"i{c['i']}k{c['k']}s{c['seed']}")
def test_gen_samplebench_matches_reference(case):
    check_samplebench(case, oracle_factory(1))  # the i = 8 seed search takes minutes on one CPU thread: GPU test


def sweep_case(case, ks, core_factory):
    al = Alphabet.default(case["n_props"])
    spec = Specification([tuple(t) for t in case["pos"]], [tuple(t) for t in case["neg"]])
    cfg = LearnerConfig(hash=HashScheme(case["hash"]), **case["cfg"])
    rows = B.run_masking_sweep(spec, al, cfg, ks, core_factory=core_factory)
    want = {r["k"]: r for r in case["rows"]}
    for r in rows:
        assert {k: r.get(k) for k in ("k", "status", "cost", "precise")} == want[r["k"]], r


@pytest.mark.parametrize("case", GOLD["masking"], ids=lambda c: c["name"])
def test_masking_sweep_rows_match_reference_subset(case):
    sweep_case(case, (1, 61, 126) if case["name"] != "simple2_k6" else (1, 126), oracle_factory(1))


def test_summarize_ruc_matches_reference_summary():
    got = B.summarize_ruc(GOLD["ruc"]["rows"])
    assert got == GOLD["ruc"]["summary"]
