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
