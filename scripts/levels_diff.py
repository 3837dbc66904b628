#!/usr/bin/env python
"""Differential check of the device-resident cost levels (levels.cuh) against the host-driven level loop on random
specifications: every case is seeded by its own index, so a mismatch is reproduced with `--only K`.
    python scripts/levels_diff.py [--cases 300] [--only K] [--first 0]"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from helpers import random_spec  # noqa: E402
from paper_2402_12373_b200 import learner as L  # noqa: E402
from paper_2402_12373_b200.scheme import HashScheme  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=300)
ap.add_argument("--first", type=int, default=0)
ap.add_argument("--only", type=int, default=-1)
a = ap.parse_args()
warnings.simplefilter("ignore")
COMBOS = [(8, 1 << 18), (8, 1 << 24), (1, 1 << 24), (4, 1 << 14), (2, 1 << 20)]
if os.environ.get("LD_COMBOS"):  # "ctas:max_work,..."
    COMBOS = [tuple(int(v) for v in c.split(":")) for c in os.environ["LD_COMBOS"].split(",")]


def summary(res):
    lv = [(x["cost"], x["offered"], x["admitted"], x["duplicates"], x["bytes"]) for x in res.stats.levels]
    return res.status, (res.text or "")[:60], res.cost, res.stats.offered, res.stats.admitted, res.stats.duplicates, lv


def records_of(spec, al, kw, opts):
    """records of every entry of a search run with LTL_CORE_OPTIONS = opts"""
    from helpers import records_array
    from paper_2402_12373_b200.core import make_core

    os.environ["LTL_CORE_OPTIONS"] = opts
    cores = []

    def factory(*x, **y):
        cores.append(make_core(*x, **y))
        real = cores[-1].close
        cores[-1].close = lambda: None
        cores[-1]._real_close = real
        return cores[-1]

    L.learn(spec, None, al, core_factory=factory, **kw)
    rec = records_array(cores[-1])
    cores[-1]._real_close()
    return rec


def explain(spec, al, kw, opts):
    a_, b_ = records_of(spec, al, kw, "device_levels=0"), records_of(spec, al, kw, opts)
    sa = {tuple(r) for r in a_.tolist()}
    extra = [(i, tuple(r)) for i, r in enumerate(b_.tolist()) if tuple(r) not in sa]
    print(f"  host entries {len(a_)}, device entries {len(b_)}, extra on the device {len(extra)}")
    if extra:
        import collections
        print("  extra by op", collections.Counter(r[0] for _, r in extra), "entry index range", extra[0][0], extra[-1][0])
        print("  first extras", extra[:12])
        print("  last extras", extra[-6:], flush=True)


bad = 0
for k in ([a.only] if a.only >= 0 else range(a.first, a.first + a.cases)):
    rng = np.random.default_rng(1000 + k)
    n_props = int(rng.integers(1, 4))
    n_pos, n_neg = int(rng.integers(1, 300)), int(rng.integers(1, 300))
    hi = int(rng.choice([5, 20, 45, 64]))
    lo = int(rng.integers(1, hi + 1))
    population = 1 << 40 if hi > 12 else sum((1 << n_props) ** length for length in range(lo, hi + 1))
    if n_pos + n_neg > population // 3:
        n_pos, n_neg = max(1, population // 8), max(1, population // 8)
    try:
        spec, al = random_spec(rng, n_props, n_pos, n_neg, lo, hi)
    except (RuntimeError, ValueError):
        continue
    kw = dict(max_cost=int(rng.integers(4, 8)))
    if rng.random() < 0.3:
        kw["noise"] = float(rng.choice([0.02, 0.1]))
    if rng.random() < 0.6:
        kw["hash"] = HashScheme(str(rng.choice(["mueller", "nh", "mueller_blocked", "fkp"])), int(rng.choice([0, 0, 20, 90])))
    if rng.random() < 0.2:
        kw["store_last_level"] = True
    if os.environ.get("LD_KW"):
        kw.update(eval(os.environ["LD_KW"]))
    os.environ["LTL_CORE_OPTIONS"] = "device_levels=0"
    want = summary(L.learn(spec, None, al, **kw))
    for ctas, mw in COMBOS:
        os.environ["LTL_CORE_OPTIONS"] = f"levels_ctas={ctas},levels_max_work={mw}"
        for rep in range(2):
            got = summary(L.learn(spec, None, al, **kw))
            if got != want:
                bad += 1
                print(f"MISMATCH case {k} ctas={ctas} max_work={mw} rep={rep} props={n_props} P={spec.n_pos} N={spec.n_neg} len={lo}..{hi} {kw}")
                print("  want", str(want)[:500])
                print("  got ", str(got)[:500], flush=True)
                explain(spec, al, kw, f"levels_ctas={ctas},levels_max_work={mw}")
                break
        else:
            if a.only >= 0:
                print(f"ok case {k} ctas={ctas} max_work={mw}", want[6][-1])
    if bad >= 5:
        break
print(f"levels_diff: {bad} mismatches")
