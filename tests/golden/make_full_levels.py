#!/usr/bin/env python
"""Per-level counters AND record hashes of the five BASELINE configurations at bench depth, from the CPU
ORACLE PORT (oracle/ltl_oracle.c, all host threads) -> tests/golden/full_levels.json.

The reference itself refuses four of the five inputs (> 64 traces or > 63 positions); the oracle is pinned
against the reference wherever the reference runs (tests/test_oracle_golden.py).  Each case records status,
formula text, cost, counters, and per cost level {offered, admitted, duplicates, bytes, entry range,
SHA-256 of the (op, lhs, rhs) records}: records determine the matrices inductively, so equal hashes mean the
same set of unique CS in the same order (north star: "same per-level count and set of unique CS").

    python tests/golden/make_full_levels.py [case ...]        (default: all; several minutes of CPU, <= 40 GB RAM)

`max_cost` of a case is the cost the planted run solves at (the level a search ends in is never stored, which is
what lets config 4 -- 16 MiB per matrix -- fit host memory); the GPU tests run the same bound.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import oracle_factory, search_with_record_hashes  # noqa: E402
from oracle import cpu_oracle  # noqa: E402
from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200.scheme import HashScheme  # noqa: E402

#: case -> (config, max_cost, budget_bytes, hash variant, random ("unsolvable") traces instead of planted ones)
CASES = {
    "c1_tiny": ("c1_tiny", 10, 2 << 30, "mueller", False),
    "c2_planted": ("c2_planted", 11, 150 << 30, "mueller", False),
    "c2_planted_mueller_blocked": ("c2_planted", 11, 150 << 30, "mueller_blocked", False),
    "c3_long": ("c3_long", 8, 150 << 30, "mueller", False),
    "c4_many": ("c4_many", 6, 4 << 40, "mueller", False),
    "c5_deep": ("c5_deep", 6, 150 << 30, "mueller", False),
    "c5_deep_budget": ("c5_deep", 8, 512 << 20, "mueller", False),  # 512 MiB budget: exhausted inside cost level 6
    "c5_random_budget": ("c5_deep", 8, 1 << 30, "mueller", True),
    "c3_random": ("c3_long", 8, 150 << 30, "mueller", True),
}

OUT = os.path.join(HERE, "full_levels.json")


def main(names):
    have = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            have = json.load(fh)
    threads = cpu_oracle.max_threads()
    for name in names:
        config, max_cost, budget, hname, rnd = CASES[name]
        wl = dict(Wl.CONFIGS[config])
        if rnd:
            spec, alphabet = Wl.random_spec(wl["n_props"], wl["n_pos"], wl["n_neg"], wl["min_len"], wl["max_len"], wl["seed"])
        else:
            spec, alphabet, _planted, wl = Wl.make_config(config)
        t0 = time.time()
        res = search_with_record_hashes(spec, alphabet, max_cost=max_cost, budget_bytes=budget,
                                        core_factory=oracle_factory(threads), hash=HashScheme(hname))
        res.update({"generator": "tests/golden/make_full_levels.py (CPU oracle port)", "config": config,
                    "workload": wl, "max_cost": max_cost, "budget_bytes": budget, "hash": hname, "random": rnd,
                    "seconds": round(time.time() - t0, 1), "threads": threads})
        have[name] = res
        print(name, res["status"], res["formula"], res["cost"], res["offered"], res["admitted"], res["seconds"], flush=True)
        with open(OUT, "w") as fh:
            json.dump(have, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
