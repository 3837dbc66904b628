"""CPU: host-side logic around the hot path -- packing, formula text/cost/overfit, suffix tables, trace files,
workload generator/evaluator, CLI plumbing -- against the reference-generated golden fixtures."""
import json
import os

import numpy as np
import pytest

from helpers import golden, oracle_factory, unhex
from paper_2402_12373_b200 import cli, workloads as Wl
from paper_2402_12373_b200.formula import CostHomomorphism, cost, overfit, overfit_cost, parse_formula, print_formula
from paper_2402_12373_b200.learner import bucket_pairs, learn
from paper_2402_12373_b200.packing import TraceContext, length_masks, rounds_for_words
from paper_2402_12373_b200.scheme import HashScheme, fkp_bits_per_row, resolve_scheme
from paper_2402_12373_b200.traces import Alphabet, Specification, SuffixTable, load_spec, save_spec


def test_length_masks_and_rounds():
    kat = golden()["kat"]["length_mask"]
    for n, want in kat.items():
        assert int(length_masks(np.array([int(n)]), 1)[0, 0]) == int(want, 16)
    for w, r in golden()["rounds_for_width"].items():
        if int(w) % 64 == 0:
            assert rounds_for_words(int(w) // 64) == r
    m = length_masks(np.array([0, 1, 64, 65, 128, 130]), 3)
    assert m[2].tolist() == [2**64 - 1, 0, 0] and m[3].tolist() == [2**64 - 1, 1 << 63, 0]
    assert m[5].tolist() == [2**64 - 1, 2**64 - 1, 3 << 62]


def test_packing_matches_reference_vectors():
    for case in golden()["opvec"]:
        traces = [tuple(t) for t in case["traces"]]
        n_pos = case["n_pos"]
        try:
            spec = Specification(traces[:n_pos], traces[n_pos:])
        except ValueError:
            continue  # the random reference vectors may repeat a trace across sides
        if spec.size != len(traces):
            continue
        ctx = TraceContext.from_spec(spec, Alphabet.default(case["n_props"]))
        assert (ctx.masks[:, 0] == unhex(case["masks"])).all()
        for p, atoms in enumerate(case["atoms"]):
            assert (ctx.atoms[p][:, 0] == unhex(atoms)).all()


def test_formula_text_cost_overfit():
    a3 = Alphabet.default(3)
    h = CostHomomorphism((1, 2, 1, 1, 3, 2, 2, 4))
    for row in golden()["formula_text"]:
        f = parse_formula(row["in"], a3)
        assert print_formula(f, a3) == row["printed"]
        assert cost(f) == row["cost"] and cost(f, h) == row["cost_w"]
        assert parse_formula(print_formula(f, a3), a3) == f
    for row in golden()["overfit"]:
        spec, al = Specification(row["pos"], row["neg"]), Alphabet.default(row["n_props"])
        assert print_formula(overfit(spec, al), al) == row["text"]
        assert overfit_cost(spec, al) == row["cost"] == cost(overfit(spec, al))
        assert overfit_cost(spec, al, h) == row["cost_w"]


def test_suffix_tables_and_scheme():
    for row in golden()["suffix"]:
        spec = Specification(row["pos"], row["neg"])
        table = SuffixTable.from_spec(spec)
        assert table.count == row["count"]
        assert list(table.rows) == row["rows"] and list(table.offsets) == row["offsets"]
        rs = resolve_scheme(HashScheme(), spec.lengths, table)
        assert rs.variant == row["variant"]
    for n, want in golden()["kat"]["fkp_bits_per_row"].items():
        assert fkp_bits_per_row(int(n)) == want


def test_bucket_pairs_follow_the_reference_rule():
    u = CostHomomorphism.uniform()
    assert bucket_pairs(u, 3, 2) == [(1, 1)]            # AND at cost 3: only (1,1)
    assert bucket_pairs(u, 6, 2) == [(1, 4), (2, 3)]    # commutative: a <= b
    assert bucket_pairs(u, 5, 7) == [(1, 3), (2, 2), (3, 1)]
    assert bucket_pairs(u, 2, 1) == [(1, None)] and bucket_pairs(u, 1, 1) == []


def test_trace_file_round_trip(tmp_path):
    spec, al, _, _ = Wl.make_config("c1_tiny")
    path = tmp_path / "t.trace"
    save_spec(spec, path, al)
    spec2, al2 = load_spec(path)
    assert spec2.pos == spec.pos and spec2.neg == spec.neg and al2.size == al.size


def test_workload_evaluator_agrees_with_the_oracle_semantics():
    """eval_formula (multi-word numpy) against the oracle's operators on nested formulas, W in {1, 3}."""
    from oracle import cpu_oracle

    rng = np.random.default_rng(0)
    for max_len in (40, 170):
        spec, al = Wl.random_spec(3, 20, 20, 5, max_len, seed=max_len)
        ctx = TraceContext.from_spec(spec, al)
        core = cpu_oracle.OracleCore(ctx.masks.reshape(-1), spec.n_pos, 0, 1, words_per_row=ctx.words)
        f = parse_formula("(p0 U (p1 & X p2)) | G(p0 | F !p2)", al)
        a = [ctx.atoms[p].reshape(-1) for p in range(3)]
        u = core.apply_binary(7, a[0], core.apply_binary(2, a[1], core.apply_unary(4, a[2])))
        g = core.apply_unary(6, core.apply_binary(3, a[0], core.apply_unary(5, core.apply_unary(1, a[2]))))
        want = core.apply_binary(3, u, g)
        assert (Wl.eval_formula(f, ctx).reshape(-1) == want).all()


def test_planted_configs_are_consistent():
    for name in ("c1_tiny", "c2_planted", "c3_long"):
        spec, al, f, cfg = Wl.make_config(name)
        assert (spec.n_pos, spec.n_neg) == (cfg["n_pos"], cfg["n_neg"])
        assert Wl.error_count(f, spec, al) == 0


def test_cli_learn_report(tmp_path, monkeypatch, capsys):
    """CLI plumbing with the learner's core factory swapped for the CPU oracle (no GPU here)."""
    spec, al, _, cfg = Wl.make_config("c1_tiny")
    path = tmp_path / "c1.trace"
    save_spec(spec, path, al)
    monkeypatch.setattr(cli, "learn", lambda *a, **kw: learn(*a, core_factory=oracle_factory(1), **kw))
    out = tmp_path / "report.json"
    rc = cli.main(["learn", str(path), "--max-cost", "10", "--json", str(out), "--verify"])
    assert rc == 0
    rep = json.loads(out.read_text())
    assert rep["status"] == "solved" and rep["formula"] == "F G p0 & (p0 U p1)" and rep["cost"] == 7
    assert rep["verified_errors"] == 0 and rep["stats"]["offered"] == 5762
    assert cli.main(["learn", str(tmp_path / "missing.trace")]) == 2


def test_specification_dedup_matches_naive_on_many_traces():
    """Hash-accelerated first-occurrence dedup and P/N clash detection (`traces.py`) against the obvious loops."""
    import warnings

    from paper_2402_12373_b200.traces import Specification

    rng = np.random.default_rng(12)
    R, L = 6000, 7
    chars = rng.integers(0, 3, size=(2 * R, L)).astype(np.uint16)   # few distinct values: thousands of duplicates
    lengths = rng.integers(0, L + 1, size=2 * R)
    lengths[:R][lengths[:R] == 0] = 1
    as_tuple = lambda k: tuple(int(c) for c in chars[k, : lengths[k]])  # noqa: E731
    pos_seen, pos = set(), []
    for k in range(R):
        t = as_tuple(k)
        if t not in pos_seen:
            pos_seen.add(t)
            pos.append(t)
    neg_seen, neg = set(), []
    for k in range(R, 2 * R):
        t = as_tuple(k)
        if t not in neg_seen and t not in pos_seen:  # keep the sides disjoint for the first check
            neg_seen.add(t)
            neg.append(t)
    keep_neg = [k for k in range(R, 2 * R) if as_tuple(k) not in pos_seen]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = Specification.from_arrays(chars[:R], lengths[:R], chars[keep_neg], lengths[keep_neg])
    assert spec.pos == tuple(pos) and spec.neg == tuple(neg)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with pytest.raises(ValueError, match="both sides"):
            Specification.from_arrays(chars[:R], lengths[:R], chars[R:], lengths[R:])


def test_array_pairs_are_a_specification_and_the_scheme_rules_take_arrays():
    """`learn` / `as_specification` accept (chars, lengths) pairs (the 10^6-trace input form); without a device they
    are the host Specification; `resolve_scheme` works on length arrays (no per-trace Python loop)."""
    from paper_2402_12373_b200.learner import as_specification
    from paper_2402_12373_b200.scheme import V_GATHER, V_MUELLER, V_NH, V_NH32

    P = [(1, 2, 3), (0, 1), (3,)]
    N = [(2, 2), (1, 0, 1, 3)]
    pc = np.array([[1, 2, 3, 9], [0, 1, 7, 7], [3, 5, 5, 5]], dtype=np.uint16)  # junk beyond the lengths
    nc = np.array([[2, 2, 0, 0], [1, 0, 1, 3]], dtype=np.uint16)
    spec = as_specification((pc, np.array([3, 2, 1])), (nc, np.array([2, 4])))
    want = Specification(P, N)
    assert spec.pos == want.pos and spec.neg == want.neg and spec.device_traces is None
    assert (spec.n_nonempty, spec.n_empty_positive, spec.max_len) == (5, 0, 4)
    assert as_specification(want, None) is want
    res = learn((pc, np.array([3, 2, 1])), (nc, np.array([2, 4])), 2, max_cost=6, core_factory=oracle_factory(1))
    assert res.text == learn(P, N, 2, max_cost=6, core_factory=oracle_factory(1)).text
    lengths = np.array([3, 2, 1, 2, 4])
    assert resolve_scheme(HashScheme(), lengths).variant == V_GATHER
    assert resolve_scheme(HashScheme(), np.full(60, 20)).variant == V_MUELLER
    assert resolve_scheme(HashScheme(), np.full(100, 20)).variant == V_NH32
    assert resolve_scheme(HashScheme(), np.full(100, 33)).variant == V_NH
    assert resolve_scheme(HashScheme("nh"), np.full(10, 32)).variant == V_NH32
