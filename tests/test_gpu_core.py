"""GPU parity tests: the CUDA screening core (through the C ABI, via ctypes) against the CPU oracle and
the reference-generated golden fixtures.  Bit-exact: matrices, records, counters, statuses, fingerprints."""
import numpy as np
import pytest

from helpers import (cfg_from_golden, golden, oracle_factory, random_spec, records_array, sha, spec_from_golden,
                     unhex)
from oracle import cpu_oracle
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200.core import CudaCore, V_FKP, V_GATHER, V_MUELLER, V_NH
from paper_2402_12373_b200.errors import CoreOOM
from paper_2402_12373_b200.formula import print_formula
from paper_2402_12373_b200.packing import length_masks

pytestmark = pytest.mark.gpu

UNARY = (1, 4, 5, 6)


@pytest.fixture(params=["compact", "tiles"])
def screen_path(request, monkeypatch):
    """Small passes over one-word rows run through the compact phase-A kernel (`k_screen_small`) by default; "tiles" forces
    them through the tile kernel (`k_screen`), which big passes always use -- every variant of it stays covered by the small
    differential cases."""
    if request.param == "tiles":
        monkeypatch.setenv("LTL_CORE_OPTIONS", "small_screen=0")
    return request.param


def assert_same_state(cuda, ora):
    assert cuda.counters() == ora._counters()
    n = ora.n_entries
    if n:
        assert (cuda.export_cms() == ora.export_cms()).all()
        assert (records_array(cuda) == records_array(ora)).all()


def make_pair(masks, n_pos, err_max=0, variant=V_MUELLER, pr=(), po=(), fkp=0, mask_k=0, budget=1 << 30, W=1, **opt):
    cuda = CudaCore(masks, n_pos, err_max, variant, pr, po, fkp, mask_k, budget, words_per_row=W, **opt)
    ora = cpu_oracle.OracleCore(masks, n_pos, err_max, variant, pr, po, fkp, mask_k, budget, words_per_row=W, threads=4)
    return cuda, ora


def random_masks(rng, R, W, full=False):
    lengths = np.full(R, 64 * W) if full else rng.integers(1, 64 * W + 1, size=R)
    return length_masks(lengths, W).reshape(-1)


def random_cm(rng, masks):
    a = rng.integers(0, 1 << 63, size=len(masks), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=len(masks), dtype=np.uint64)
    return a & masks


def drive(cuda, ora, rng, n_seed=5, rounds=2):
    """Same call sequence on both cores; every return value must agree."""
    masks = ora_masks = None  # noqa
    for k in range(n_seed):
        cm = random_cm(rng, drive.masks)
        assert cuda.add_entry(cm, 0, k, -1) == ora.add_entry(cm, 0, k, -1)
    lo = 0
    for _ in range(rounds):
        hi = ora.n_entries
        for op in UNARY:
            assert cuda.screen_unary(op, lo, hi) == ora.screen_unary(op, lo, hi)
        for op, tri in ((2, True), (3, True), (7, False)):
            assert cuda.screen_binary(op, 0, hi, 0, hi, tri) == ora.screen_binary(op, 0, hi, 0, hi, tri)
        mid = ora.n_entries
        assert cuda.screen_binary(7, hi, mid, 0, hi, False) == ora.screen_binary(7, hi, mid, 0, hi, False)
        assert cuda.screen_binary(2, 1, hi, 0, mid, True) == ora.screen_binary(2, 1, hi, 0, mid, True)
        lo = hi
        if ora.n_entries > 6000:
            break


@pytest.mark.parametrize("R,W", [(2, 1), (16, 1), (64, 1), (65, 1), (200, 1), (1024, 1), (7, 2), (33, 3), (20, 4),
                                 (9, 5), (12, 7), (40, 8), (5, 11), (24, 16), (130, 16)])
@pytest.mark.parametrize("variant", [V_MUELLER, V_NH], ids=["mueller", "nh"])
def test_differential_random(R, W, variant, screen_path):
    rng = np.random.default_rng(1000 * R + W)
    masks = random_masks(rng, R, W)
    n_pos = int(rng.integers(1, R)) if R > 1 else 1
    cuda, ora = make_pair(masks, n_pos, err_max=-1, variant=variant, W=W)  # err_max -1: nothing ever solves
    drive.masks = masks
    drive(cuda, ora, rng, n_seed=4, rounds=2 if R * W <= 2048 else 1)
    assert_same_state(cuda, ora)
    cm = random_cm(rng, masks)
    assert cuda.fingerprint_of(cm) == ora.fingerprint_of(cm)
    assert cuda.contains(cm) == ora.contains(cm)
    e = ora.get_cm(ora.n_entries // 2)
    assert cuda.contains(e) and ora.contains(e)
    assert (cuda.get_cm(ora.n_entries // 2) == e).all()
    assert cuda.get_record(3) == ora.get_record(3)
    cuda.close()


@pytest.mark.parametrize("R,W,split,chunk", [(200, 1, 3, 97), (1024, 1, 16, 1000), (130, 16, 2, 333), (64, 3, 1, 50),
                                             (300, 2, 4, 1 << 20)])
@pytest.mark.parametrize("variant", [V_MUELLER, V_NH], ids=["mueller", "nh"])
def test_differential_split_and_chunked(R, W, split, chunk, variant, screen_path):
    """Row-split evaluation (partial fingerprints combined by atomics) and tiny chunks (rows cut mid-way)."""
    rng = np.random.default_rng(77 * R + W)
    masks = random_masks(rng, R, W)
    cuda, ora = make_pair(masks, R // 2, err_max=-1, variant=variant, W=W, chunk_candidates=chunk)
    cuda.set_option("force_split", split)
    drive.masks = masks
    drive(cuda, ora, rng, n_seed=4, rounds=1)
    assert_same_state(cuda, ora)
    cuda.close()


@pytest.mark.parametrize("seed", range(6))
def test_solver_and_counters(seed, screen_path):
    """First solver in enumeration order wins; counters stop at the solver (reference _speedups.pyx:372-374)."""
    rng = np.random.default_rng(500 + seed)
    R, W = (24, 1) if seed % 2 == 0 else (12, 2)
    masks = random_masks(rng, R, W)
    n_pos = R // 2
    err_max = R // 2 - 2 - seed % 3  # loose enough that something solves early
    cuda, ora = make_pair(masks, n_pos, err_max=err_max, W=W, chunk_candidates=[1 << 20, 64][seed % 2])
    drive.masks = masks
    for k in range(4):
        cm = random_cm(rng, masks)
        assert cuda.add_entry(cm, 0, k, -1) == ora.add_entry(cm, 0, k, -1)
    statuses = []
    lo = 0
    for _ in range(3):
        hi = ora.n_entries
        for op in UNARY:
            a, b = cuda.screen_unary(op, lo, hi), ora.screen_unary(op, lo, hi)
            assert a == b
            statuses.append(a[0])
        for op, tri in ((2, True), (3, True), (7, False)):
            a, b = cuda.screen_binary(op, 0, hi, 0, hi, tri), ora.screen_binary(op, 0, hi, 0, hi, tri)
            assert a == b
            statuses.append(a[0])
        assert_same_state(cuda, ora)
        lo = hi
    assert 1 in statuses, "test should exercise the SOLVED path"
    cuda.close()


def test_budget_oom_matches_oracle(screen_path):
    rng = np.random.default_rng(9)
    R = 32
    masks = random_masks(rng, R, 1)
    eb = 8 * R + 16
    for cap in (1, 3, 10, 57):
        cuda, ora = make_pair(masks, 16, err_max=-1, budget=cap * eb + 5, chunk_candidates=40)
        for k in range(5):
            cm = random_cm(rng, masks)
            try:
                want = ora.add_entry(cm, 0, k, -1)
            except cpu_oracle.CoreOOM:
                with pytest.raises(CoreOOM):
                    cuda.add_entry(cm, 0, k, -1)
                continue
            assert cuda.add_entry(cm, 0, k, -1) == want
        n0 = ora.n_entries
        for op in UNARY:
            assert cuda.screen_unary(op, 0, n0) == ora.screen_unary(op, 0, n0)
        assert cuda.screen_binary(7, 0, n0, 0, n0, False) == ora.screen_binary(7, 0, n0, 0, n0, False)
        assert_same_state(cuda, ora)
        cuda.close()


def test_fingerprint_golden():
    for case in golden()["fpvec"]:
        cuda = CudaCore(unhex(case["masks"]), 1, 0, case["variant"], case["proj_rows"], case["proj_offs"],
                        case["fkp_bits"], case["mask_k"])
        for cm, fp in zip(case["cms"], case["fps"]):
            assert cuda.fingerprint_of(unhex(cm)) == int(fp, 16)
        cuda.close()


def test_operator_golden_vectors():
    names = {1: "not", 2: "and", 3: "or", 4: "next", 5: "finally", 6: "globally", 7: "until"}
    for case in golden()["opvec"]:
        masks = unhex(case["masks"])
        cuda = CudaCore(masks, case["n_pos"], -1, V_MUELLER)
        x, y = unhex(case["x"]), unhex(case["y"])
        assert cuda.add_entry(x, 0, 0, -1) == 0
        iy = cuda.add_entry(y, 0, 1, -1)
        if iy < 0:
            cuda.close()
            continue
        for op in UNARY:
            cuda.screen_unary(op, 0, 1)
        for op in (2, 3, 7):
            cuda.screen_binary(op, 0, 1, 1, 2, False)
        op_arr, lhs, rhs = cuda.export_records()
        cms = cuda.export_cms()
        for e in range(2, len(op_arr)):
            assert (cms[e] == unhex(case[names[int(op_arr[e])]])).all(), names[int(op_arr[e])]
        cuda.close()


def test_transcripts_golden():
    from test_oracle_golden import _replay_transcript

    for tr in golden()["transcripts"]:
        cuda = CudaCore(unhex(tr["masks"]), tr["n_pos"], 0, V_MUELLER, budget_bytes=1 << 24)
        _replay_transcript(cuda, tr)
        assert cuda.counters() == tr["counters"]
        assert sha(cuda.export_cms()) == tr["cms_sha"]
        assert sha(records_array(cuda)) == tr["records_sha"]
        cuda.close()


@pytest.mark.parametrize("native_loop,options", [(True, ""), (False, ""), (True, "small_screen=0,small_admit=0"),
                                                 (True, "device_levels=0"), (True, "levels_ctas=1"),
                                                 (True, "levels_max_work=2048")],
                         ids=["run_search", "run_level", "big_kernels", "host_levels", "levels_one_cta", "levels_hand_over"])
@pytest.mark.parametrize("case", golden()["learn"], ids=lambda c: c["name"])
def test_learn_golden_cases(case, native_loop, options, monkeypatch):
    """The product path end to end (learner -> C ABI -> CUDA) against the reference's recorded outcomes, with the
    cost-level loop inside the library (`ltl_core_run_search`, the default: the first small levels in one launch planned
    on the device, `levels.cuh`, the rest host-driven), with that launch switched off, on one CTA, handing over to the
    host-driven path early, and with one `run_level` call per level from `learner.py`."""
    monkeypatch.setattr(L.Enumeration, "native_loop", native_loop)
    if options:  # small passes through the kernels big passes use (tile phase A, four bookkeeping kernels)
        monkeypatch.setenv("LTL_CORE_OPTIONS", options)
    spec, alphabet = spec_from_golden(case)
    cfg = cfg_from_golden(case["cfg"])
    cores = []
    from paper_2402_12373_b200.core import make_core

    def factory(*a, **kw):
        cores.append(make_core(*a, **kw))
        real_close = cores[-1].close
        cores[-1].close = lambda: None
        cores[-1]._real_close = real_close
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
    if "core" in case and cores:
        core, g = cores[-1], case["core"]
        assert core.n_entries == g["n_entries"]
        assert sha(core.export_cms()) == g["cms_sha"]
        assert sha(records_array(core)) == g["records_sha"]
    for c in cores:
        c._real_close()


@pytest.mark.parametrize("n_props,n_pos,n_neg,length,max_cost,chunk", [
    (3, 512, 512, 64, 6, None),      # BASELINE config 2 shape (one full word per trace)
    (3, 256, 256, 1024, 4, None),    # BASELINE config 3 shape (16 words per row)
    (3, 40, 40, 200, 5, 5000),       # 4 words per row, chunked
    (5, 100, 100, 64, 4, None),
])
def test_learn_matches_oracle_beyond_reference_limits(n_props, n_pos, n_neg, length, max_cost, chunk):
    rng = np.random.default_rng(n_props * 1000 + n_pos)
    spec, alphabet = random_spec(rng, n_props, n_pos, n_neg, length, length)
    want = L.learn(spec, None, alphabet, max_cost=max_cost, core_factory=oracle_factory(8), overfit_on_ceiling=False,
                   budget_bytes=8 << 30)
    opts = {} if chunk is None else {"chunk_candidates": chunk}
    from paper_2402_12373_b200.core import make_core

    cores = []

    def factory(*a, **kw):
        cores.append(make_core(*a, **kw, **opts))
        rc = cores[-1].close
        cores[-1].close = lambda: None
        cores[-1]._real_close = rc
        return cores[-1]

    got = L.learn(spec, None, alphabet, max_cost=max_cost, core_factory=factory, overfit_on_ceiling=False,
                  budget_bytes=8 << 30)
    assert got.status == want.status
    assert got.text == want.text and got.cost == want.cost
    a, b = got.stats.as_dict(), want.stats.as_dict()
    for lv in a["levels"] + b["levels"]:
        lv.pop("ms", None)
    assert a == b
    for c in cores:
        c._real_close()


@pytest.mark.parametrize("variant", [V_MUELLER, V_NH], ids=["mueller", "nh"])
def test_many_rows_row_split(variant):
    """BASELINE config 4 shape, scaled: many short traces => row-split evaluation with combined fingerprints."""
    rng = np.random.default_rng(4)
    R = 1 << 14
    masks = random_masks(rng, R, 1)
    cuda, ora = make_pair(masks, R // 2, err_max=-1, variant=variant, budget=4 << 30)
    drive.masks = masks
    for k in range(4):
        cm = random_cm(rng, masks)
        assert cuda.add_entry(cm, 0, k, -1) == ora.add_entry(cm, 0, k, -1)
    n0 = ora.n_entries
    for op in UNARY:
        assert cuda.screen_unary(op, 0, n0) == ora.screen_unary(op, 0, n0)
    n1 = ora.n_entries
    assert cuda.screen_binary(2, 0, n1, 0, n1, True) == ora.screen_binary(2, 0, n1, 0, n1, True)
    assert cuda.screen_binary(7, 0, n0, 0, n1, False) == ora.screen_binary(7, 0, n0, 0, n1, False)
    assert cuda.counters() == ora._counters()
    hi, lo = cuda.entry_fingerprints()
    for e in (0, n0, ora.n_entries - 1):
        assert (int(hi[e]) << 64 | int(lo[e])) == ora.fingerprint_of(ora.get_cm(e))
        assert (cuda.get_cm(e) == ora.get_cm(e)).all()
    assert sha(cuda.export_cms()) == sha(ora.export_cms())
    cuda.close()


def test_argument_errors():
    masks = np.full(4, 2**64 - 1, dtype=np.uint64)
    with pytest.raises(ValueError):
        CudaCore(masks, 1, 0, V_GATHER, list(range(127)), [0] * 127)
    with pytest.raises(ValueError):
        CudaCore(masks, 1, 0, V_MUELLER, words_per_row=17)
    core = CudaCore(masks, 2, 0, V_MUELLER)
    with pytest.raises(ValueError):
        core.add_entry(np.zeros(3, dtype=np.uint64), 0, 0, -1)
    with pytest.raises(IndexError):
        core.get_cm(0)
    with pytest.raises(ValueError):
        core.screen_unary(1, 0, 5)
    core.close()


def test_last_level_matrices_can_be_skipped():
    """store_results=0 (what the learner does on the final cost level): identical statuses, counters and
    records, but the skipped matrices cannot be read or used as operands."""
    rng = np.random.default_rng(31)
    masks = random_masks(rng, 40, 1)
    cuda, ora = make_pair(masks, 20, err_max=-1)
    drive.masks = masks
    for k in range(4):
        cm = random_cm(rng, masks)
        assert cuda.add_entry(cm, 0, k, -1) == ora.add_entry(cm, 0, k, -1)
    n0 = ora.n_entries
    for op in UNARY:
        assert cuda.screen_unary(op, 0, n0) == ora.screen_unary(op, 0, n0)
    n1 = ora.n_entries
    cuda.set_option("store_results", 0)
    assert cuda.screen_binary(7, 0, n1, 0, n1, False) == ora.screen_binary(7, 0, n1, 0, n1, False)
    assert cuda.counters() == ora._counters()
    assert (records_array(cuda) == records_array(ora)).all()
    assert (cuda.export_cms(0, n1) == ora.export_cms(0, n1)).all()
    with pytest.raises((ValueError, IndexError)):
        cuda.get_cm(n1)
    with pytest.raises(ValueError):
        cuda.screen_unary(1, n1, n1 + 1)
    cuda.close()


def test_fused_unary_levels_match_unfused(screen_path):
    """run_level fuses the unary connectives of a level into one pass per operand group; same results as
    screening them one at a time."""
    from paper_2402_12373_b200.learner import Segment

    rng = np.random.default_rng(32)
    masks = random_masks(rng, 100, 1)
    a, b = (CudaCore(masks, 50, -1, V_MUELLER) for _ in range(2))
    b.set_option("fuse_unary", 0)
    for k in range(5):
        cm = random_cm(rng, masks)
        assert a.add_entry(cm, 0, k, -1) == b.add_entry(cm, 0, k, -1)
    lo = 0
    for _ in range(2):
        hi = a.n_entries
        segs = [Segment(1, lo, hi), Segment(2, 0, hi, 0, hi, True), Segment(4, lo, hi), Segment(5, lo, hi),
                Segment(6, lo, hi), Segment(7, 0, hi, 0, hi, False)]
        assert a.run_level(segs) == b.run_level(segs)
        assert a.counters() == b.counters()
        lo = hi
    assert (a.export_cms() == b.export_cms()).all()
    assert (records_array(a) == records_array(b)).all()
    a.close()
    b.close()


@pytest.mark.parametrize("sub_tiles,chunk", [(8, None), (16, 700), (64, None)])
def test_sub_launched_levels_match_oracle(sub_tiles, chunk):
    """Phase A issued in many small launches (early stop after a solver) gives the sequential result."""
    rng = np.random.default_rng(sub_tiles)
    spec, alphabet = random_spec(rng, 2, 20, 20, 10, 30)
    want = L.learn(spec, None, alphabet, max_cost=9, core_factory=oracle_factory(4))
    from paper_2402_12373_b200.core import make_core

    def factory(*a, **kw):
        core = make_core(*a, **kw, **({} if chunk is None else {"chunk_candidates": chunk}))
        core.set_option("sub_tiles", sub_tiles)
        return core

    got = L.learn(spec, None, alphabet, max_cost=9, core_factory=factory)
    assert (got.status, got.text, got.cost) == (want.status, want.text, want.cost)
    a, b = got.stats.as_dict(), want.stats.as_dict()
    for lv in a["levels"] + b["levels"]:
        lv.pop("ms", None)
    assert a == b


@pytest.mark.parametrize("tiled", [0, 1])
@pytest.mark.parametrize("R,W", [(64, 1), (300, 2), (40, 16)])
def test_both_phase_b_forms_match_oracle(tiled, R, W):
    """Phase B from records (one warp per 32 new entries) and tile-shaped (phase A's tiles + verdicts)."""
    from paper_2402_12373_b200.learner import Segment

    rng = np.random.default_rng(R + W + tiled)
    masks = random_masks(rng, R, W)
    cuda, ora = make_pair(masks, R // 2, err_max=-1, variant=V_NH if tiled else V_MUELLER, W=W)
    cuda.set_option("tiled_materialize", tiled)
    drive.masks = masks
    for k in range(5):
        cm = random_cm(rng, masks)
        assert cuda.add_entry(cm, 0, k, -1) == ora.add_entry(cm, 0, k, -1)
    lo = 0
    for _ in range(2):
        hi = ora.n_entries
        segs = [Segment(1, lo, hi), Segment(2, 0, hi, 0, hi, True), Segment(3, 0, hi, 0, hi, True), Segment(4, lo, hi),
                Segment(5, lo, hi), Segment(6, lo, hi), Segment(7, 0, hi, 0, hi, False)]
        st = cuda.run_level(segs)
        for s in segs:
            got = ora.screen_unary(s.op, s.a0, s.a1) if s.unary else ora.screen_binary(s.op, s.a0, s.a1, s.b0, s.b1, s.tri)
            assert got[0] == 0
        assert st[0] == 0
        lo = hi
        if ora.n_entries > 3000:
            break
    assert_same_state(cuda, ora)
    cuda.close()


@pytest.mark.parametrize("R,L,n_props,W", [(1, 1, 1, 1), (37, 5, 2, 1), (200, 64, 3, 1), (64, 63, 16, 1), (50, 100, 5, 2),
                                           (33, 1024, 3, 16), (9, 700, 7, 11), (5000, 32, 4, 1), (20, 130, 9, 4)])
def test_device_packing_matches_host_packing(R, L, n_props, W):
    """k_pack (reference bitsem.py:73-88 on the device) against the np.packbits path, ragged lengths, empty rows."""
    from paper_2402_12373_b200.core import pack_traces
    from paper_2402_12373_b200.packing import TraceContext
    from paper_2402_12373_b200.traces import Alphabet, Specification

    rng = np.random.default_rng(R * 31 + L)
    lengths = rng.integers(1, L + 1, size=R).astype(np.int64)
    if R > 3:
        lengths[-1] = 0  # an empty (negative) trace
        lengths[0] = L
    chars = rng.integers(0, 1 << n_props, size=(R, L)).astype(np.uint16)  # junk beyond the lengths must be ignored
    masks, atoms = pack_traces(chars, lengths, n_props, W)
    clean = chars.copy()
    clean[np.arange(L)[None, :] >= lengths[:, None]] = 0
    spec = Specification.__new__(Specification)
    spec._chars, spec._lengths, spec.n_pos, spec.n_neg = clean, lengths, max(R - 1, 1), R - max(R - 1, 1)
    want = TraceContext.from_spec(spec, Alphabet.default(n_props), words=W)
    assert (masks == want.masks).all()
    assert (atoms == want.atoms).all()


@pytest.mark.parametrize("R,err_max,budget_entries,chunk", [(16, -1, None, None), (64, -1, None, None), (100, -1, None, None),
                                                            (200, -1, None, None), (1024, -1, None, None),
                                                            (100, 40, None, None), (64, 27, None, None),
                                                            (100, -1, 700, None), (130, -1, None, 500), (256, 110, None, 3000),
                                                            (200, -1, None, 6), (256, -1, None, 7)])  # pass = the fused NOTs only
@pytest.mark.parametrize("variant", [V_MUELLER, V_NH], ids=["mueller", "nh"])
@pytest.mark.parametrize("kernels", ["small", "tiles"])
def test_fused_not_levels_match_unfused(R, err_max, budget_entries, chunk, variant, kernels):
    """Phase B of a level also screens NOT(new entry) for the next level (k_materialize_not): identical statuses,
    counters, matrices and records to screening NOT in a pass of its own -- with partial 64-row fingerprint blocks,
    a solver among the fused candidates, the budget running out inside them, and chunks that cut the NOT unit.
    Where the solver rank is final after a tile has run (tile kernels without row split: "tiles" forces that for every
    R) the fused launch goes out behind the tiles of the AND / OR segments, which do not read the new entries, and stores
    only if they found no solver (`gate_store`): core `c` keeps round 1's order, and the read-back at the end writes what
    a closed gate left pending."""
    from paper_2402_12373_b200.learner import Segment

    rng = np.random.default_rng(9000 + R)
    masks = random_masks(rng, R, 1)
    budget = (1 << 40) if budget_entries is None else budget_entries * (8 * R + 16)
    kw = {} if chunk is None else {"chunk_candidates": chunk}
    a, b, c = (CudaCore(masks, R // 2, err_max, variant, budget_bytes=budget, **kw) for _ in range(3))
    a.set_option("fuse_not_min", 0)  # by default only launches that fill the device are fused
    a.set_option("gate_store", 1)
    c.set_option("fuse_not_min", 0)
    c.set_option("gate_store", 0)
    b.set_option("fuse_not", 0)
    if kernels == "tiles":
        for core in (a, c):
            core.set_option("small_screen", 0)
            core.set_option("max_split", 1)
    for k in range(5):
        cm = random_cm(rng, masks)
        assert a.add_entry(cm, 0, k, -1) == b.add_entry(cm, 0, k, -1) == c.add_entry(cm, 0, k, -1)
    lo = 0
    expect_skip = 0
    for level in range(3):
        hi = a.n_entries
        if hi > 200:  # the next level would have millions of entries
            break
        segs = [Segment(1, lo, hi), Segment(2, 0, hi, 0, hi, True), Segment(3, 0, hi, 0, hi, True), Segment(4, lo, hi),
                Segment(5, lo, hi), Segment(6, lo, hi), Segment(7, 0, hi, 0, hi, False)]
        ra, rb, rc = a.run_level(segs), b.run_level(segs), c.run_level(segs)
        assert ra == rb == rc
        assert a.counters() == b.counters() == c.counters()
        if ra[0] != 0:
            # solved behind the NOT segment of a whole-level pass whose NOTs were fused (level 0 reads imported atoms)
            # (... and in front of the first segment that reads the new entries: NEXT, index 3)
            if ra[0] == 1 and ra[1] < 3 and level > 0 and chunk is None and kernels == "tiles":
                expect_skip = 1 if ra[1] > 0 else None  # (a solving NOT may hide a solver behind it that closed the gate)
            break
        lo = hi
    assert c.info()["gated_skips"] == 0 and a.info()["gated_skips"] == (expect_skip if expect_skip is not None else a.info()["gated_skips"])
    want = b.export_cms()
    assert (a.export_cms() == want).all() and (c.export_cms() == want).all()
    assert (records_array(a) == records_array(b)).all() and (records_array(c) == records_array(b)).all()
    for core in (a, b, c):
        core.close()


def test_deadline_interrupts_a_level_between_passes():
    """The reference checks its deadline between the chunks of a level (`enumerator.py:278`, `290`); here a level is one
    library call, so the core checks it between its passes (`deadline_ms`, status LTL_S_TIMEOUT): a search whose last
    level alone takes seconds is abandoned shortly after the deadline, not at the end of the level; what earlier passes
    admitted stays admitted, and a deadline that never fires changes nothing."""
    import time

    from paper_2402_12373_b200 import workloads as Wl
    from paper_2402_12373_b200.errors import TimeoutExceeded
    from paper_2402_12373_b200.learner import S_TIMEOUT, Segment, learn

    spec, alphabet = Wl.random_spec(3, 512, 512, 64, 64, 77)  # nothing solves: every level is exhaustive
    free = learn(spec, None, alphabet, max_cost=8)
    timed = learn(spec, None, alphabet, max_cost=8, deadline_s=600.0)  # armed, never fires: smaller passes, same result
    assert (timed.status, timed.stats.offered, timed.stats.admitted) == (free.status, free.stats.offered, free.stats.admitted)
    assert [(r["cost"], r["offered"], r["admitted"]) for r in timed.stats.levels] == \
        [(r["cost"], r["offered"], r["admitted"]) for r in free.stats.levels]
    t0 = time.monotonic()
    with pytest.raises(TimeoutExceeded):
        # cost levels up to 10 take ~5 ms, level 11 (12 M candidates, six passes with a deadline armed) ~15 ms
        learn(spec, None, alphabet, max_cost=13, deadline_s=0.01, budget_bytes=100 << 30)
    assert time.monotonic() - t0 < 1.0
    # on the core itself: the status, and the entries of the passes that ran
    masks = np.full(1024, ~np.uint64(0), dtype=np.uint64)
    core = CudaCore(masks, 512, -1, V_NH, budget_bytes=8 << 30)
    rng = np.random.default_rng(5)
    for k in range(3):
        assert core.add_entry(rng.integers(0, 1 << 63, size=1024, dtype=np.uint64), 0, k, -1) == k
    assert core.run_level([Segment(2, 0, 3, 0, 3, False)])[0] == 0
    core.set_option("chunk_candidates", 4)
    core.set_option("deadline_ms", 1)
    time.sleep(0.01)
    n0 = core.n_entries
    assert core.run_level([Segment(3, 0, n0, 0, n0, False)])[0] == S_TIMEOUT and core.n_entries == n0
    core.set_option("deadline_ms", 0)
    assert core.run_level([Segment(3, 0, n0, 0, n0, False)])[0] == 0 and core.n_entries > n0
    core.close()


def test_debug_mask_invariant(monkeypatch):
    """The reference's LTLLEARN_DEBUG_MASKS assertion (`bitsem.py:46-61`: no characteristic bit outside the validity
    mask after any operation) on the device: with the variable set (or option ``debug_masks``) every matrix the core
    stores is checked -- a whole search over ragged traces passes unchanged, a bad matrix is refused."""
    from paper_2402_12373_b200.learner import learn

    spec, alphabet = random_spec(np.random.default_rng(91), 2, 70, 70, 0, 90)  # ragged lengths, two words per row
    plain = learn(spec, None, alphabet, max_cost=6)
    monkeypatch.setenv("LTLLEARN_DEBUG_MASKS", "1")
    checked = learn(spec, None, alphabet, max_cost=6)
    assert (checked.status, checked.text, checked.stats.offered, checked.stats.admitted) == \
        (plain.status, plain.text, plain.stats.offered, plain.stats.admitted)
    half, al3 = random_spec(np.random.default_rng(92), 3, 90, 90, 0, 30)       # half-width store
    assert learn(half, None, al3, max_cost=5).stats.admitted > 0
    monkeypatch.delenv("LTLLEARN_DEBUG_MASKS")
    masks = length_masks(np.array([5, 64, 0, 17]), 1).reshape(-1)
    core = CudaCore(masks, 2, -1, V_MUELLER)
    ok = np.array([0xF8 << 56, 1, 0, 1 << 63], dtype=np.uint64) & masks
    bad = ok.copy()
    bad[2] = 1 << 40  # a bit in an empty trace
    assert core.add_entry(bad, 0, 0, -1) == 0  # unchecked by default, like the reference
    core.set_option("debug_masks", 1)
    assert core.add_entry(ok, 0, 1, -1) == 1
    with pytest.raises(AssertionError, match="escaped the validity mask"):
        core.add_entry(bad ^ np.uint64(1 << 41), 0, 2, -1)
    core.close()


@pytest.mark.parametrize("R,W,variant,fuse_not_min", [(64, 1, V_NH, 1), (200, 1, V_MUELLER, 1 << 30), (100, 2, V_NH, 1), (40, 16, V_NH, 1)])
def test_phase_b_order_matches_oracle(R, W, variant, fuse_not_min):
    """Phase B walks big right-operand buckets block by block (`k_mat_plan`: runs of consecutive new entries found from
    the winner flags, processed as "for each block of j: all i"); the entries, their order and their matrices are those
    of the entry-order walk.  Forced onto small levels here: blocks of 32 entries, every pass planned."""
    from paper_2402_12373_b200.learner import Segment

    rng = np.random.default_rng(R * 3 + W)
    masks = random_masks(rng, R, W)
    cuda, ora = make_pair(masks, R // 2, err_max=-1, variant=variant, W=W)
    plain = CudaCore(masks, R // 2, -1, variant, words_per_row=W)
    for name, value in (("small_admit", 0), ("order_min", 1), ("order_block_bytes", 8 * R * W * 32), ("fuse_not_min", fuse_not_min)):
        cuda.set_option(name, value)
    plain.set_option("order_mat", 0)
    for k in range(6):
        cm = random_cm(rng, masks)
        assert cuda.add_entry(cm, 0, k, -1) == ora.add_entry(cm, 0, k, -1) == plain.add_entry(cm, 0, k, -1)
    lo = 0
    for _ in range(3):
        hi = ora.n_entries
        segs = [Segment(1, lo, hi), Segment(2, 0, hi, 0, hi, True), Segment(3, 0, lo, lo, hi, False), Segment(4, lo, hi),
                Segment(5, lo, hi), Segment(6, lo, hi), Segment(7, 0, hi, 0, hi, False), Segment(7, 0, 3, 0, hi, False)]
        segs = [s for s in segs if s.a1 > s.a0 and (s.unary or s.b1 > s.b0)]
        st = cuda.run_level(segs)
        assert plain.run_level(segs) == st
        for s in segs:
            got = ora.screen_unary(s.op, s.a0, s.a1) if s.unary else ora.screen_binary(s.op, s.a0, s.a1, s.b0, s.b1, s.tri)
            assert got[0] == 0
        assert st[0] == 0
        lo = hi
        if ora.n_entries > 4000:
            break
    assert ora.n_entries > 300
    assert_same_state(cuda, ora)
    assert (plain.export_cms() == cuda.export_cms()).all()
    cuda.close()
    plain.close()


@pytest.mark.gpu
def test_device_levels_match_host_levels(monkeypatch):
    """The device-resident first levels (`levels.cuh`: one launch, planned on the device) against the host-driven level
    loop on random specifications -- rows in one and in several hash blocks, every fingerprint variant, masking, noise,
    a stored and an unstored last level -- for several cluster sizes and hand-over points.  The cases share one process
    on purpose: cores are built on pooled arenas, and what an earlier search left in them (partial sums beyond the part
    small passes clear) once leaked into the next one."""
    from paper_2402_12373_b200.scheme import HashScheme

    def summary(res):
        lv = [(x["cost"], x["offered"], x["admitted"], x["duplicates"], x["bytes"]) for x in res.stats.levels]
        return res.status, res.text, res.cost, res.stats.offered, res.stats.admitted, res.stats.duplicates, lv

    for k in range(60):
        rng = np.random.default_rng(1000 + k)
        n_props = int(rng.integers(1, 4))
        n_pos, n_neg = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        hi = int(rng.choice([5, 20, 45, 64]))
        lo = int(rng.integers(1, hi + 1))
        population = 1 << 40 if hi > 12 else sum((1 << n_props) ** length for length in range(lo, hi + 1))
        if n_pos + n_neg > population // 3:
            n_pos, n_neg = max(1, population // 8), max(1, population // 8)
        try:
            spec, alphabet = random_spec(rng, n_props, n_pos, n_neg, lo, hi)
        except (RuntimeError, ValueError):
            continue
        kw = dict(max_cost=int(rng.integers(4, 8)))
        if rng.random() < 0.3:
            kw["noise"] = float(rng.choice([0.02, 0.1]))
        if rng.random() < 0.6:
            kw["hash"] = HashScheme(str(rng.choice(["mueller", "nh", "mueller_blocked", "fkp"])), int(rng.choice([0, 0, 20, 90])))
        if rng.random() < 0.2:
            kw["store_last_level"] = True
        monkeypatch.setenv("LTL_CORE_OPTIONS", "device_levels=0")
        want = summary(L.learn(spec, None, alphabet, **kw))
        for ctas, max_work in ((8, 1 << 18), (8, 1 << 24), (1, 1 << 24), (4, 1 << 14)):
            monkeypatch.setenv("LTL_CORE_OPTIONS", f"levels_ctas={ctas},levels_max_work={max_work}")
            assert summary(L.learn(spec, None, alphabet, **kw)) == want, (k, ctas, max_work, kw)
