"""CPU: the multi-GPU orchestration (candidate-range sharding, hash-owner all-to-all, ordered admission,
record all-gather) with world_size 2 over gloo processes and with 3 virtual ranks on threads, against the
single-core CPU oracle.  The device stages are replaced by tests/stage_oracle.py."""
import os
import sys
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import oracle_factory, random_spec
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200.sharded import ThreadComm, TorchComm, owner_of, sharded_core_factory
from stage_oracle import OracleStageCore

CASES = [
    dict(seed=11, n_props=2, n_pos=6, n_neg=6, lo=3, hi=9, kw=dict(max_cost=8)),
    dict(seed=12, n_props=3, n_pos=10, n_neg=9, lo=4, hi=12, kw=dict(max_cost=6)),
    dict(seed=13, n_props=2, n_pos=8, n_neg=8, lo=6, hi=14, kw=dict(max_cost=7, budget_bytes=150 * (16 * 8 + 16) + 3)),
    dict(seed=14, n_props=2, n_pos=7, n_neg=7, lo=5, hi=10, kw=dict(max_cost=7, require_nnf=True)),
]


def _summary(res):
    lv = [(x["cost"], x["offered"], x["admitted"], x["duplicates"], x["bytes"]) for x in res.stats.levels]
    return res.status, res.text, res.cost, res.stats.offered, res.stats.admitted, res.stats.duplicates, lv


def _reference(case):
    spec, alphabet = random_spec(np.random.default_rng(case["seed"]), case["n_props"], case["n_pos"], case["n_neg"],
                                 case["lo"], case["hi"])
    return spec, alphabet, _summary(L.learn(spec, None, alphabet, core_factory=oracle_factory(1), **case["kw"]))


def _sharded(case, comm):
    spec, alphabet = random_spec(np.random.default_rng(case["seed"]), case["n_props"], case["n_pos"], case["n_neg"],
                                 case["lo"], case["hi"])
    factory = sharded_core_factory(comm, local_factory=OracleStageCore)
    return _summary(L.learn(spec, None, alphabet, core_factory=factory, **case["kw"]))


def _gloo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        got = [_sharded(case, comm) for case in CASES]
        out.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_sharded_learn_world2_gloo():
    want = [_reference(case)[2] for case in CASES]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = 29500 + os.getpid() % 2000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(out.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert any(w[0] == "oom" for w in want) and any(w[0] == "solved" for w in want)
    for rank in (0, 1):
        assert results[rank] == want, f"rank {rank}"


@pytest.mark.parametrize("world", [3, 4])
def test_sharded_learn_virtual_ranks(world):
    comms = ThreadComm.group(world)
    for case in CASES[:3]:
        want = _reference(case)[2]
        got, errs = [None] * world, []

        def work(r):
            try:
                got[r] = _sharded(case, comms[r])
            except BaseException as exc:  # noqa: BLE001
                errs.append(exc)
                comms[r]._s.barrier.abort()

        threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errs, errs
        assert all(g == want for g in got)


def test_owner_function_is_balanced_and_deterministic():
    g = torch.Generator().manual_seed(1)
    fp = torch.randint(-(1 << 62), 1 << 62, (20000, 2), generator=g, dtype=torch.int64)
    for world in (2, 3, 8):
        o = owner_of(fp, world)
        assert int(o.min()) >= 0 and int(o.max()) < world
        counts = torch.bincount(o, minlength=world).float()
        assert float(counts.max() / counts.min()) < 1.15
        assert torch.equal(o, owner_of(fp.clone(), world))


# ------------------------------------------------------------------------------------------------ row shards (host logic)


def test_row_slices_cut_on_fingerprint_blocks():
    from paper_2402_12373_b200.sharded import row_slices

    assert row_slices(1024, 1, 8) == [(128 * g, 128 * (g + 1)) for g in range(8)]
    assert row_slices(512, 16, 8) == [(64 * g, 64 * (g + 1)) for g in range(8)]      # 16 words per row: 4-row units
    assert row_slices(170, 1, 2) == [(0, 128), (128, 170)]                           # only the last shard is short
    assert row_slices(1 << 21, 1, 8)[-1] == (7 << 18, 1 << 21)
    for n_rows, W, G in [(1024, 1, 8), (300, 3, 2), (8192, 1, 4), (100, 16, 4), (515, 5, 3)]:
        sl = row_slices(n_rows, W, G)
        assert sl[0][0] == 0 and sl[-1][1] == n_rows and all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        assert all((a * W) % 64 == 0 for a, _ in sl)
    with pytest.raises(ValueError):
        row_slices(100, 1, 4)     # 64-row blocks: the third and fourth shard would be empty
    with pytest.raises(ValueError):
        row_slices(24, 3, 2)


class _FakeLocal:
    """Records what RowShardedCore hands to its local core."""

    def __init__(self, n_words):
        self.n, self.entries = n_words, []

    def add_entry(self, cm, op, lhs, rhs):
        assert len(cm) == self.n
        self.entries.append(np.array(cm, dtype=np.uint64))
        return len(self.entries) - 1

    def get_cm(self, idx):
        return self.entries[idx].copy()

    def contains(self, cm):
        return any((cm == e).all() for e in self.entries)

    def counters(self):
        return len(self.entries), 0, 0, 0, 0


def _row_worker(comm, n_rows, W, out):
    from paper_2402_12373_b200.sharded import RowShardedCore, row_slices

    import torch

    r0, r1 = row_slices(n_rows, W, comm.world)[comm.rank]
    core = RowShardedCore(_FakeLocal((r1 - r0) * W), comm, r0, r1, n_rows, W)
    rng = np.random.default_rng(11)
    cms = [rng.integers(0, 1 << 63, size=n_rows * W, dtype=np.uint64) for _ in range(3)]
    for k, cm in enumerate(cms):
        assert core.add_entry(cm, 0, k, -1) == k
    assert (core.local.entries[1] == cms[1][r0 * W: r1 * W]).all()          # each shard keeps its rows only
    gathered = [core.get_cm(k) for k in range(3)]                           # ... and get_cm puts them back together
    assert all((g == c).all() for g, c in zip(gathered, cms))
    assert core.contains(cms[2]) and core.n_entries == 3
    # the exchange: wrapping sums, every rank ends with the same totals
    big = torch.tensor([(1 << 63) - 1, -5, 7 + comm.rank], dtype=torch.int64)
    small = torch.tensor([2**31 - 1, comm.rank], dtype=torch.int32)
    comm.all_reduce_sum([big, small])
    out.append((comm.rank, big.tolist(), small.tolist()))


def _expected_sums(world):
    wrap64 = lambda v: (v + (1 << 63)) % (1 << 64) - (1 << 63)  # noqa: E731
    wrap32 = lambda v: (v + (1 << 31)) % (1 << 32) - (1 << 31)  # noqa: E731
    return ([wrap64(world * ((1 << 63) - 1)), -5 * world, sum(7 + r for r in range(world))],
            [wrap32(world * (2**31 - 1)), sum(range(world))])


@pytest.mark.parametrize("world,n_rows,W", [(2, 170, 1), (3, 400, 3), (4, 256, 16)])
def test_row_sharded_wrapper_virtual_ranks(world, n_rows, W):
    comms = ThreadComm.group(world)
    out, errs = [], []

    def work(r):
        try:
            _row_worker(comms[r], n_rows, W, out)
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            comms[r]._s.barrier.abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    assert len(out) == world and all((b, s) == _expected_sums(world) for _, b, s in out)


def _gloo_row_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        _row_worker(TorchComm(), 170, 1, out)
        q.put(out[0])
    finally:
        dist.destroy_process_group()


def test_row_sharded_wrapper_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 2000
    procs = [ctx.Process(target=_gloo_row_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(r for r, _, _ in results) == [0, 1]
    assert all((b, s) == _expected_sums(2) for _, b, s in results)


# ------------------------------------------------------------------------------------------------ row shards (whole searches)

ROW_CASES = [
    dict(seed=41, n_props=2, n_pos=100, n_neg=70, lo=5, hi=40, kw=dict(max_cost=6)),                     # solved or ceiling
    dict(seed=42, n_props=2, n_pos=30, n_neg=110, lo=70, hi=130, kw=dict(max_cost=5)),                   # 3 words per row
    dict(seed=43, n_props=2, n_pos=90, n_neg=90, lo=10, hi=64, kw=dict(max_cost=6, budget_bytes=150 * (180 * 8 + 16) + 1)),
    dict(seed=44, n_props=3, n_pos=64, n_neg=64, lo=3, hi=20, kw=dict(max_cost=6, noise=0.1)),           # errors summed
    dict(seed=45, n_props=2, n_pos=80, n_neg=80, lo=6, hi=30, kw=dict(max_cost=8), planted="F(p0 & X p1)"),  # solved
    dict(seed=46, n_props=2, n_pos=70, n_neg=90, lo=6, hi=30, kw=dict(max_cost=8, noise=0.3), planted="G(p0 | X p1)"),
]


def _row_case_spec(case):
    if "planted" in case:
        from paper_2402_12373_b200 import workloads as Wl

        spec, alphabet, _ = Wl.planted_spec(case["n_props"], case["n_pos"], case["n_neg"], case["lo"], case["hi"],
                                            case["planted"], case["seed"])
        return spec, alphabet
    return random_spec(np.random.default_rng(case["seed"]), case["n_props"], case["n_pos"], case["n_neg"], case["lo"],
                       case["hi"])


def _row_sharded(case, comm):
    from paper_2402_12373_b200.sharded import row_sharded_core_factory
    from stage_oracle import OracleRowShard

    spec, alphabet = _row_case_spec(case)
    factory = row_sharded_core_factory(comm, local_factory=OracleRowShard)
    return _summary(L.learn(spec, None, alphabet, core_factory=factory, **case["kw"]))


def _gloo_rows_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        out.put((rank, [_row_sharded(case, comm) for case in ROW_CASES]))
    except BaseException as exc:  # the parent must not wait for its timeout when a rank dies
        out.put((rank, f"{type(exc).__name__}: {exc}"))
        raise
    finally:
        dist.destroy_process_group()


def test_row_sharded_learn_world2_gloo():
    """Whole searches over two row shards (gloo processes, CPU stand-in shards): the exchange of per-candidate sums
    and the replicated admission reproduce the single oracle core -- formula, counters, per-level rows."""
    want = []
    for case in ROW_CASES:
        spec, alphabet = _row_case_spec(case)
        want.append(_summary(L.learn(spec, None, alphabet, core_factory=oracle_factory(1), **case["kw"])))
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = 33500 + os.getpid() % 2000
    procs = [ctx.Process(target=_gloo_rows_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(out.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert any(w[0] == "oom" for w in want) and any(w[0] == "solved" for w in want)
    for rank in (0, 1):
        assert results[rank] == want, f"rank {rank}"
