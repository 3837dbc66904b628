"""GPU parity of the half-width store (variant NH32: traces of at most 32 positions are kept two rows per 64-bit
word, north-star "uint32 words"): the CUDA core against the CPU oracle -- matrices cross the C ABI as uint64[R]
either way, so every comparison is on the reference's own layout.  Bit-exact."""
import threading

import numpy as np
import pytest

from helpers import oracle_factory, random_spec, records_array, search_with_record_hashes
from oracle import cpu_oracle
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200.core import CudaCore, V_NH32
from paper_2402_12373_b200.packing import length_masks
from paper_2402_12373_b200.scheme import HashScheme, V_NH32 as S_NH32, resolve_scheme

pytestmark = pytest.mark.gpu

UNARY = (1, 4, 5, 6)


def short_masks(rng, R, full=False):
    lengths = np.full(R, 32) if full else rng.integers(1, 33, size=R)
    return length_masks(lengths, 1).reshape(-1)


def random_cm(rng, masks):
    return (rng.integers(0, 1 << 32, size=len(masks), dtype=np.uint64) << np.uint64(32)) & masks


def drive(cuda, ora, rng, masks, n_seed=4, rounds=2):
    for k in range(n_seed):
        cm = random_cm(rng, masks)
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
        lo = hi
        if ora.n_entries > 6000:
            break


def same_state(cuda, ora):
    assert cuda.counters() == ora._counters()
    assert (cuda.export_cms() == ora.export_cms()).all()
    assert (records_array(cuda) == records_array(ora)).all()


@pytest.mark.parametrize("R,n_pos", [(2, 1), (3, 1), (3, 2), (64, 31), (65, 32), (129, 64), (129, 65), (200, 1), (200, 199),
                                     (1024, 512), (1025, 513), (4097, 2000)])
def test_differential_random(R, n_pos):
    rng = np.random.default_rng(31 * R + n_pos)
    masks = short_masks(rng, R)
    cuda = CudaCore(masks, n_pos, -1, V_NH32)
    ora = cpu_oracle.OracleCore(masks, n_pos, -1, cpu_oracle.V_NH32, threads=4)
    drive(cuda, ora, rng, masks, rounds=2 if R <= 2048 else 1)
    same_state(cuda, ora)
    cm = random_cm(rng, masks)
    assert cuda.fingerprint_of(cm) == ora.fingerprint_of(cm)
    assert cuda.contains(cm) == ora.contains(cm)
    e = ora.get_cm(ora.n_entries // 2)
    assert cuda.contains(e) and (cuda.get_cm(ora.n_entries // 2) == e).all()
    cuda.close()


@pytest.mark.parametrize("R,split,chunk", [(300, 2, 97), (1024, 8, 1000), (1025, 3, 333), (5000, 16, 1 << 20)])
def test_split_and_chunked(R, split, chunk):
    rng = np.random.default_rng(7 * R)
    masks = short_masks(rng, R)
    cuda = CudaCore(masks, R // 2, -1, V_NH32, chunk_candidates=chunk)
    cuda.set_option("force_split", split)
    ora = cpu_oracle.OracleCore(masks, R // 2, -1, cpu_oracle.V_NH32, threads=4)
    drive(cuda, ora, rng, masks, rounds=1)
    same_state(cuda, ora)
    cuda.close()


@pytest.mark.parametrize("seed", range(8))
def test_solver_errors_and_noise(seed):
    """The verdict bits of both halves: first solver in order, counters cut at the solver, with odd / even n_pos."""
    rng = np.random.default_rng(900 + seed)
    R = [70, 71, 200, 333][seed % 4]
    n_pos = R // 2 + seed % 2
    masks = short_masks(rng, R)
    err_max = R // 2 - 3 - seed % 3
    cuda = CudaCore(masks, n_pos, err_max, V_NH32, chunk_candidates=[1 << 20, 64][seed % 2])
    ora = cpu_oracle.OracleCore(masks, n_pos, err_max, cpu_oracle.V_NH32, threads=2)
    for k in range(4):
        cm = random_cm(rng, masks)
        assert cuda.add_entry(cm, 0, k, -1) == ora.add_entry(cm, 0, k, -1)
    lo = 0
    for _ in range(3):
        hi = ora.n_entries
        done = False
        for op in UNARY:
            a, b = cuda.screen_unary(op, lo, hi), ora.screen_unary(op, lo, hi)
            assert a == b
            done |= a[0] != 0
        for op, tri in ((2, True), (3, True), (7, False)):
            a, b = cuda.screen_binary(op, 0, hi, 0, hi, tri), ora.screen_binary(op, 0, hi, 0, hi, tri)
            assert a == b
            done |= a[0] != 0
        assert cuda.counters() == ora._counters()
        lo = hi
        if done:
            break
    cuda.close()


@pytest.mark.parametrize("n_props,n_pos,n_neg,lo,hi,max_cost,chunk", [
    (2, 40, 41, 3, 32, 7, None), (3, 100, 99, 20, 32, 6, None), (2, 300, 301, 1, 32, 7, 5000), (3, 700, 500, 32, 32, 6, None),
    (2, 33, 32, 1, 12, 8, 1000)])
def test_learn_matches_oracle(n_props, n_pos, n_neg, lo, hi, max_cost, chunk):
    rng = np.random.default_rng(n_pos * 7 + n_neg)
    spec, alphabet = random_spec(rng, n_props, n_pos, n_neg, lo, hi)
    assert resolve_scheme(HashScheme(), spec.lengths).variant == S_NH32
    want = search_with_record_hashes(spec, alphabet, max_cost=max_cost, budget_bytes=1 << 30, core_factory=oracle_factory(4))

    def factory(*a, **kw):
        from paper_2402_12373_b200.core import make_core

        return make_core(*a, **kw, **({"chunk_candidates": chunk} if chunk else {}))

    got = search_with_record_hashes(spec, alphabet, max_cost=max_cost, budget_bytes=1 << 30, core_factory=factory)
    assert got == want
    # and a noisy run: error counts over both halves decide the solver
    a = L.learn(spec, None, alphabet, max_cost=max_cost, noise=0.2, core_factory=oracle_factory(4), overfit_on_ceiling=False)
    b = L.learn(spec, None, alphabet, max_cost=max_cost, noise=0.2, overfit_on_ceiling=False)
    assert (a.status, a.text, a.cost, a.stats.offered, a.stats.admitted) == (b.status, b.text, b.cost, b.stats.offered, b.stats.admitted)


def test_fused_not_levels():
    """Phase B with the next level's NOT fused in, on the half-width store (forced onto small levels)."""
    rng = np.random.default_rng(3)
    spec, alphabet = random_spec(rng, 2, 150, 151, 8, 32)
    want = search_with_record_hashes(spec, alphabet, max_cost=8, budget_bytes=1 << 30, core_factory=oracle_factory(4))

    def factory(*a, **kw):
        from paper_2402_12373_b200.core import make_core

        core = make_core(*a, **kw)
        core.set_option("fuse_not_min", 1)
        return core

    assert search_with_record_hashes(spec, alphabet, max_cost=8, budget_bytes=1 << 30, core_factory=factory) == want


@pytest.mark.parametrize("world", [2, 3])
def test_row_shards(world):
    """Row shards of the half-width store: shard boundaries at multiples of 128 rows."""
    from paper_2402_12373_b200.sharded import ThreadComm, row_sharded_core_factory, row_slices

    rng = np.random.default_rng(11 + world)
    spec, alphabet = random_spec(rng, 2, 300, 333, 4, 32)
    assert all(a % 128 == 0 for a, _ in row_slices(spec.size, 1, world, half_width=True))
    want = search_with_record_hashes(spec, alphabet, max_cost=7, budget_bytes=1 << 30, core_factory=oracle_factory(4))
    comms = ThreadComm.group(world)
    got, errs = [None] * world, []

    def work(r):
        try:
            got[r] = search_with_record_hashes(spec, alphabet, max_cost=7, budget_bytes=1 << 30,
                                               core_factory=row_sharded_core_factory(comms[r]))
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            comms[r]._s.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for res in got:
        assert res == want
