#!/usr/bin/env python
"""Randomised differential soak on a GPU box: random specifications / options, the CUDA core (single, fused NOT forced
on small levels, row-sharded over thread ranks) against the CPU oracle -- status, formula text, cost, counters and
per-level rows must be identical.  `python scripts/soak.py --seconds 600 [--seed 1]`; exits 1 on the first mismatch."""
import argparse
import os
import sys
import threading
import time
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from helpers import oracle_factory, random_spec  # noqa: E402
from paper_2402_12373_b200 import learner as L  # noqa: E402
from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200.scheme import HashScheme  # noqa: E402
from paper_2402_12373_b200.sharded import ThreadComm, row_sharded_core_factory, row_slices, sharded_core_factory  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=300)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--big", action="store_true", help="up to 3000 traces per specification, shallower searches")
a = ap.parse_args()
warnings.simplefilter("ignore")
if os.environ.get("SOAK_ONLY"):
    import faulthandler

    faulthandler.dump_traceback_later(45, repeat=False, file=sys.stdout)
FORMULAS = ["p0 U (p1 & X p0)", "F (p0 & X p1)", "G (p0 | X p1)", "(p0 U p1) & F G p0", "X X p1 | G p0", "!p0 & F p1"]


def W_ALL(spec):
    return -(-spec.max_len // 64)


def summary(res):
    lv = [(x["cost"], x["offered"], x["admitted"], x["duplicates"], x["bytes"]) for x in res.stats.levels]
    return res.status, res.text, res.cost, res.stats.offered, res.stats.admitted, res.stats.duplicates, lv


def threaded(world, make, spec, al, kw):
    comms = ThreadComm.group(world)
    got, errs = [None] * world, []

    def work(r):
        try:
            got[r] = summary(L.learn(spec, None, al, core_factory=make(comms[r]), **kw))
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            comms[r]._s.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    [t.start() for t in ts]
    deadline = time.time() + 120
    [t.join(max(0.0, deadline - time.time())) for t in ts]
    if any(t.is_alive() for t in ts):
        print("HANG", world, make.__name__, [t.is_alive() for t in ts], flush=True)
        os._exit(3)
    if errs:
        raise errs[0]
    return got


rng = np.random.default_rng(a.seed)
t_end, n = time.time() + a.seconds, 0
while time.time() < t_end:
    n += 1
    n_props = int(rng.integers(1, 4))
    top = 1500 if a.big else 200
    n_pos, n_neg = int(rng.integers(1, top)), int(rng.integers(1, top))
    hi = int(rng.choice([5, 20, 63, 64, 65, 130, 200]))
    lo = int(rng.integers(1, hi + 1))
    population = 1 << 40 if hi > 12 else sum((1 << n_props) ** length for length in range(lo, hi + 1))
    if n_pos + n_neg > population // 3:  # not enough distinct traces of these lengths
        n_pos, n_neg = max(1, population // 8), max(1, population // 8)
    planted = rng.random() < 0.5 and n_props >= 2
    try:
        if planted:
            spec, al, _ = Wl.planted_spec(n_props, n_pos, n_neg, lo, hi, str(rng.choice(FORMULAS)), int(rng.integers(1 << 30)))
        else:
            spec, al = random_spec(rng, n_props, n_pos, n_neg, lo, hi)
    except (RuntimeError, ValueError):
        continue
    kw = dict(max_cost=int(rng.integers(4, 7 if a.big else 8)))
    if rng.random() < 0.3:
        kw["noise"] = float(rng.choice([0.02, 0.1, 0.3]))
    if rng.random() < 0.2:
        kw["require_nnf"] = True
    if rng.random() < 0.2:
        kw["forbid_until"] = True
    if rng.random() < 0.25:
        kw["budget_bytes"] = int(rng.integers(50, 3000)) * (8 * spec.size * -(-spec.max_len // 64) + 16) + 1
    if rng.random() < 0.2:
        kw["hash"] = HashScheme(str(rng.choice(["mueller", "nh", "mueller_blocked", "fkp"])), int(rng.choice([0, 0, 20, 90])))
    desc = f"#{n} props={n_props} P={spec.n_pos} N={spec.n_neg} len={lo}..{hi} planted={planted} {kw}"
    fused_opts = "fuse_not_min=0" + (",chunk_candidates=%d" % int(rng.integers(100, 5000)) if rng.random() < 0.3 else "")
    # the fused launch behind phase A with its store gated on the solver (needs passes without row split), or round 1's order
    fused_opts += str(rng.choice([",gate_store=1,small_screen=0,max_split=1", ",gate_store=1,max_split=1", ",gate_store=1", ",gate_store=0"]))
    with_cand2 = rng.random() < 0.3
    if os.environ.get("SOAK_ONLY") and n > int(os.environ["SOAK_ONLY"]):
        break
    if os.environ.get("SOAK_ONLY") and n != int(os.environ["SOAK_ONLY"]):
        continue
    if os.environ.get("SOAK_VERBOSE"):
        print("start", desc, flush=True)
    want = summary(L.learn(spec, None, al, core_factory=oracle_factory(8), **kw))
    if os.environ.get("SOAK_VERBOSE"):
        print("  oracle", want[0], (want[1] or "")[:60], want[2], want[3], flush=True)
    runs = {}
    os.environ.pop("LTL_CORE_OPTIONS", None)
    runs["single"] = [summary(L.learn(spec, None, al, **kw))]
    os.environ["LTL_CORE_OPTIONS"] = fused_opts
    runs["fused"] = [summary(L.learn(spec, None, al, **kw))]
    # the device-resident first levels (levels.cuh) switched off; and on a smaller cluster, handing over to the
    # host-driven path at a random point
    os.environ["LTL_CORE_OPTIONS"] = "device_levels=0"
    runs["host_levels"] = [summary(L.learn(spec, None, al, **kw))]
    os.environ["LTL_CORE_OPTIONS"] = "levels_ctas=%d,levels_max_work=%d" % (int(rng.choice([1, 2, 4, 8])), int(rng.choice([1 << 10, 1 << 14, 1 << 18, 1 << 24])))
    if os.environ.get("SOAK_LEVELS_OPTS"):  # reproduction of one case with chosen options
        os.environ["LTL_CORE_OPTIONS"] = os.environ["SOAK_LEVELS_OPTS"]
    runs["levels_hand_over"] = [summary(L.learn(spec, None, al, **kw))]
    # round 2 paths: the level loop driven from Python (one run_level per level) with the big-pass bookkeeping kernels and
    # the phase-B order forced onto every pass (blocks of 32 entries); the specification uploaded as array pairs and
    # checked / packed / searched on the device; the reference's debug invariant on every stored matrix
    n_words = spec.size * W_ALL(spec)
    os.environ["LTL_CORE_OPTIONS"] = f"small_admit=0,order_min=1,order_block_bytes={8 * n_words * 32}" + (",fuse_not_min=0" if rng.random() < 0.5 else "")
    L.Enumeration.native_loop = False
    try:
        runs["pyloop_ordered"] = [summary(L.learn(spec, None, al, **kw))]
    finally:
        L.Enumeration.native_loop = True
    os.environ.pop("LTL_CORE_OPTIONS", None)
    P_arr = (spec.chars[: spec.n_pos].copy(), spec.lengths[: spec.n_pos].copy())
    N_arr = (spec.chars[spec.n_pos:].copy(), spec.lengths[spec.n_pos:].copy())
    os.environ["LTLLEARN_DEBUG_MASKS"] = "1"
    L.DEVICE_SPEC_MIN_CHARS = 0  # the device-resident path whatever the size
    try:
        runs["arrays_debug"] = [summary(L.learn(P_arr, N_arr, al, **kw))]
    finally:
        os.environ.pop("LTLLEARN_DEBUG_MASKS", None)
    hashed = kw.get("hash", HashScheme()).variant != "fkp" and want is not None
    W = -(-spec.max_len // 64)
    for world in (2, 3):
        try:
            row_slices(spec.size, W, world)
        except ValueError:
            continue
        # row shards need a block-combinable fingerprint: not the exact "gather" mode of tiny specifications, not fkp
        if hashed and spec.size * W > 64 + 62:
            try:
                if os.environ.get("SOAK_VERBOSE"):
                    print("  rows", world, flush=True)
                runs[f"rows{world}"] = threaded(world, row_sharded_core_factory, spec, al, kw)
            except ValueError as exc:
                if "block-combinable" not in str(exc):
                    raise
    os.environ.pop("LTL_CORE_OPTIONS", None)
    if with_cand2:
        if os.environ.get("SOAK_VERBOSE"):
            print("  cand2", flush=True)
        runs["cand2"] = threaded(2, sharded_core_factory, spec, al, kw)
    bad = [(k, g) for k, gs in runs.items() for g in gs if g != want]
    if bad:
        short = lambda g: (g[0], (g[1] or "")[:80], g[2:])  # noqa: E731
        print("MISMATCH", desc)
        print(" want", short(want))
        for k, g in bad:
            print(" got ", k, short(g))
        sys.exit(1)
    if n % 20 == 0:
        print(f"{n} cases ok; last: {desc} -> {want[0]} {want[1]!r} [{', '.join(runs)}]", flush=True)
print(f"soak ok: {n} cases in {a.seconds:.0f} s")
