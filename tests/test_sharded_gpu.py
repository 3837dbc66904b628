"""GPU: the sharded path with G virtual ranks on threads of one process, every rank a real `CudaCore` on
cuda:0 (its own table shard, its own replica of the store), against the single-core CUDA path and the CPU
oracle.  Exercises stage_eval / stage_file / stage_decode / stage_append / stage_purge through the C ABI."""
import threading

import numpy as np
import pytest

from helpers import oracle_factory, random_spec
from paper_2402_12373_b200 import learner as L
from paper_2402_12373_b200.sharded import ThreadComm, sharded_core_factory

pytestmark = pytest.mark.gpu


def _summary(res):
    lv = [(x["cost"], x["offered"], x["admitted"], x["duplicates"], x["bytes"]) for x in res.stats.levels]
    return res.status, res.text, res.cost, res.stats.offered, res.stats.admitted, res.stats.duplicates, lv


def _run_sharded(world, spec, alphabet, kw, **options):
    comms = ThreadComm.group(world)
    got, errs = [None] * world, []

    def work(r):
        try:
            got[r] = _summary(L.learn(spec, None, alphabet, core_factory=sharded_core_factory(comms[r], **options), **kw))
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
