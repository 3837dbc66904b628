"""GPU: the sharded path with G virtual ranks on threads of one process, every rank a real `CudaCore` on
cuda:0 (its own table shard, its own replica of the store), against the single-core CUDA path and the CPU
oracle.  Exercises stage_eval / stage_file / stage_decode / stage_append / stage_purge through the C ABI."""
import threading

import numpy as np
import pytest

from helpers import oracle_factory, random_spec
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200.sharded import ThreadComm, row_sharded_core_factory, row_slices, sharded_core_factory

pytestmark = pytest.mark.gpu


def _summary(res):
    lv = [(x["cost"], x["offered"], x["admitted"], x["duplicates"], x["bytes"]) for x in res.stats.levels]
    return res.status, res.text, res.cost, res.stats.offered, res.stats.admitted, res.stats.duplicates, lv


def _run_sharded(world, spec, alphabet, kw, make_factory=sharded_core_factory, **options):
    comms = ThreadComm.group(world)
    got, errs = [None] * world, []

    def work(r):
        try:
            got[r] = _summary(L.learn(spec, None, alphabet, core_factory=make_factory(comms[r], **options), **kw))
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            comms[r]._s.barrier.abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    return got


@pytest.mark.parametrize("world,n_props,n_pos,n_neg,lo,hi,kw", [
    (2, 2, 10, 10, 8, 20, dict(max_cost=9)),
    (3, 3, 20, 20, 30, 63, dict(max_cost=7)),
    (4, 2, 16, 16, 10, 30, dict(max_cost=8, budget_bytes=900 * (32 * 8 + 16) + 1)),
    (2, 3, 100, 100, 64, 64, dict(max_cost=6)),
    (8, 2, 12, 12, 100, 130, dict(max_cost=7)),          # 3 words per row
])
def test_sharded_matches_single_core_and_oracle(world, n_props, n_pos, n_neg, lo, hi, kw):
    spec, alphabet = random_spec(np.random.default_rng(world * 100 + n_pos), n_props, n_pos, n_neg, lo, hi)
    want = _summary(L.learn(spec, None, alphabet, core_factory=oracle_factory(4), **kw))
    single = _summary(L.learn(spec, None, alphabet, **kw))
    assert single == want
    for got in _run_sharded(world, spec, alphabet, kw):
        assert got == want


def test_sharded_stage_eval_slices_cover_the_level():
    """Arbitrary rank slices of a level (cut inside rows, inside triangular pieces) give the same fingerprints
    as the whole level."""
    import torch

    from paper_2402_12373_b200.core import CudaCore, V_MUELLER
    from paper_2402_12373_b200.learner import Segment
    from paper_2402_12373_b200.packing import length_masks

    rng = np.random.default_rng(5)
    R = 70
    masks = length_masks(rng.integers(1, 65, size=R), 1).reshape(-1)
    core = CudaCore(masks, R // 2, -1, V_MUELLER)
    for k in range(9):
        cm = (rng.integers(0, 1 << 63, size=R, dtype=np.uint64) * np.uint64(2)) & masks
        core.add_entry(cm, 0, k, -1)
    n = core.n_entries
    segs = [Segment(1, 0, n), Segment(2, 0, n, 0, n, True), Segment(3, 2, n, 0, n - 1, True), Segment(4, 0, n),
            Segment(7, 0, n, 0, n, False), Segment(7, 1, 4, 2, n, False)]
    total = core.level_size(segs)
    full, _ = core.stage_eval(segs, 0, total)
    for cuts in ([0, 1, 2, total], [0, 7, 33, 34, 100, total], list(range(0, total, 13)) + [total]):
        parts = [core.stage_eval(segs, a, b)[0] for a, b in zip(cuts[:-1], cuts[1:])]
        assert torch.equal(torch.cat(parts, 0), full)
    ranks = torch.arange(total, dtype=torch.int64, device=full.device)
    op, lhs, rhs = core.stage_decode(segs, ranks)
    # the decoded records enumerate the segments in the reference order
    from stage_oracle import seg_candidates

    want = [c for s in segs for c in seg_candidates(s)]
    assert [tuple(int(v) for v in t) for t in zip(op.tolist(), lhs.tolist(), rhs.tolist())] == want
    core.close()


def test_bench_sharded_path_runs_under_torchrun_nccl():
    """The N > 1 arm of bench.py (torchrun, NCCL process group, hash-owner all-to-all) on the one GPU a test box
    has: world size 1 forced through the sharded path; same formula as the single-core arm."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LTL_FORCE_SHARDED="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
           "--master-port", "29541", os.path.join(root, "bench.py"), "--gpus", "1", "--steps", "2", "--warmup", "3",
           "--config", "c1_tiny"]
    res = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    line = [l for l in res.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 1 and d["formula"] == "F G p0 & (p0 U p1)" and d["cost"] == 7
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.parametrize("world,n_props,n_pos,n_neg,lo,hi,kw", [
    (2, 2, 64, 64, 8, 20, dict(max_cost=7)),                       # 128 rows: one 64-word block per shard
    (2, 3, 100, 70, 30, 63, dict(max_cost=6)),                     # last shard short, partial last block; n_pos inside shard 1
    (4, 2, 200, 300, 10, 64, dict(max_cost=6)),                    # shards 0,1 hold positives only / mixed; 3 hold negatives only
    (3, 2, 150, 150, 20, 64, dict(max_cost=7, budget_bytes=700 * (300 * 8 + 16) + 1)),  # budget runs out (whole-matrix bytes)
    (2, 2, 90, 100, 100, 130, dict(max_cost=6)),                   # 3 words per row: shards are multiples of 64 rows
    (4, 3, 256, 256, 64, 64, dict(max_cost=7, noise=0.05)),        # a noisy solver: error counts are summed across shards
    (2, 2, 2048, 2048, 40, 64, dict(max_cost=6)),                  # big enough for the fused NOT in phase B on every shard
])
def test_row_sharded_matches_single_core_and_oracle(world, n_props, n_pos, n_neg, lo, hi, kw, monkeypatch):
    """G row shards (each a real CudaCore on cuda:0 over its slice of the rows, partial sums added through the
    exchange callback) reproduce the single core and the CPU oracle: status, formula, counters, per-level rows."""
    if n_pos >= 256:  # also run the fused NOT of phase B (normally only on launches that fill the device) on shards
        monkeypatch.setenv("LTL_CORE_OPTIONS", "fuse_not_min=0")
    spec, alphabet = random_spec(np.random.default_rng(world * 1000 + n_pos), n_props, n_pos, n_neg, lo, hi)
    try:
        row_slices(spec.size, -(-spec.max_len // 64), world)
    except ValueError:
        pytest.skip("too few rows for this many shards")
    want = _summary(L.learn(spec, None, alphabet, core_factory=oracle_factory(8), **kw))
    single = _summary(L.learn(spec, None, alphabet, **kw))
    assert single == want
    # with the uniqueness table sharded by fingerprint owner (the default: winner flags OR-ed over the shards) and with a
    # replica of the whole table on every shard
    for shard_table in (True, False):
        for got in _run_sharded(world, spec, alphabet, kw, make_factory=row_sharded_core_factory, shard_table=shard_table):
            assert got == want, shard_table


def test_row_sharded_matrices_and_membership():
    """get_cm gathers the rows of an entry from the shards; contains / fingerprint_of are collective."""
    from paper_2402_12373_b200.core import CudaCore, V_NH
    from paper_2402_12373_b200.learner import Segment
    from paper_2402_12373_b200.packing import length_masks

    rng = np.random.default_rng(77)
    R, world = 192, 3
    masks = length_masks(rng.integers(1, 65, size=R), 1).reshape(-1)
    seeds = [(rng.integers(0, 1 << 63, size=R, dtype=np.uint64) * np.uint64(2)) & masks for _ in range(6)]
    ref = CudaCore(masks, 80, -1, V_NH)
    for k, cm in enumerate(seeds):
        ref.add_entry(cm, 0, k, -1)
    n = ref.n_entries
    segs = [Segment(1, 0, n), Segment(2, 0, n, 0, n, True), Segment(7, 0, n, 0, n, False)]
    ref.run_level(segs)
    comms = ThreadComm.group(world)
    out, errs = [None] * world, []

    def work(r):
        try:
            core = row_sharded_core_factory(comms[r])(masks, 80, -1, V_NH, (), (), 0, 0, 2 << 30)
            for k, cm in enumerate(seeds):
                core.add_entry(cm, 0, k, -1)
            st = core.run_level(segs)
            probe = ref.get_cm(ref.n_entries - 1)
            out[r] = (st, core.counters(), [core.get_cm(i).tolist() for i in (0, n, core.n_entries - 1)],
                      core.contains(probe), core.contains(probe ^ masks), core.fingerprint_of(probe),
                      [core.get_record(i) for i in range(core.n_entries)])
            core.close()
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            comms[r]._s.barrier.abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    probe = ref.get_cm(ref.n_entries - 1)
    want = ((0, -1, -1, -1), ref.counters(), [ref.get_cm(i).tolist() for i in (0, n, ref.n_entries - 1)], True,
            ref.contains(probe ^ masks), ref.fingerprint_of(probe), [ref.get_record(i) for i in range(ref.n_entries)])
    for got in out:
        assert got == want
    ref.close()


@pytest.mark.parametrize("sharding", ["rows", "candidates"])
def test_cli_learn_under_torchrun(tmp_path, sharding):
    """`torchrun -m paper_2402_12373_b200.cli learn` (one process per GPU): process group of size 1 forced through the
    sharded cores; the report is the single-core one."""
    import json
    import os
    import subprocess
    import sys

    from paper_2402_12373_b200 import workloads as Wl
    from paper_2402_12373_b200.traces import save_spec

    spec, al, _, _ = Wl.make_config("c1_tiny")
    path, out = tmp_path / "c1.trace", tmp_path / "report.json"
    save_spec(spec, path, al)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LTL_FORCE_SHARDED="1", PYTHONPATH=root)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
           "--master-port", "29547", "-m", "paper_2402_12373_b200.cli", "learn", str(path), "--max-cost", "10", "--json",
           str(out), "--verify", "--sharding", sharding]
    res = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    rep = json.loads(out.read_text())
    assert rep["status"] == "solved" and rep["formula"] == "F G p0 & (p0 U p1)" and rep["cost"] == 7
    assert rep["verified_errors"] == 0 and rep["stats"]["offered"] == 5762


@pytest.mark.parametrize("n,world", [(0, 2), (1, 1), (1, 3), (31, 2), (1025, 8), (5000, 3), (70000, 8), (4096, 64)])
def test_stage_route_and_winners_match_the_tensor_formulation(n, world):
    """`ltl_core_stage_route` (stable counting sort of (hi, lo, rank) tuples by hash owner) and `ltl_core_stage_winners`
    (verdict bytes -> ascending winner ranks) against the tensor formulation they replace (stable sort by `owner_of`,
    scatter, nonzero)."""
    import torch

    from paper_2402_12373_b200.core import CudaCore, V_NH
    from paper_2402_12373_b200.sharded import owner_of

    core = CudaCore(np.full(4, ~np.uint64(0), dtype=np.uint64), 2, -1, V_NH)
    g = torch.Generator().manual_seed(n * 131 + world)
    fp = torch.randint(-(1 << 62), 1 << 62, (n, 2), generator=g, dtype=torch.int64).cuda()
    rank_base, level_lo = 10_000_000_019, 777
    send, counts = core.stage_route(fp, rank_base, world)
    owner = owner_of(fp, world)
    order = torch.sort(owner, stable=True)[1] if n else torch.zeros(0, dtype=torch.int64, device="cuda")
    want = torch.cat([fp[order], (rank_base + torch.arange(n, dtype=torch.int64, device="cuda"))[order].unsqueeze(1)], 1)
    assert counts == [int((owner == d).sum()) for d in range(world)] and sum(counts) == n
    assert torch.equal(send, want)
    win = (torch.rand(n, generator=g) < 0.4).to(torch.uint8).cuda()
    got = core.stage_winners(send, win, rank_base, level_lo)
    want_ranks = torch.sort(send[:, 2][win.bool()] - rank_base + level_lo)[0]
    assert torch.equal(got, want_ranks)
    core.close()
