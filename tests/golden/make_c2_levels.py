#!/usr/bin/env python
"""Per-level counts of the bench workload (BASELINE config 2, full size) from the CPU ORACLE PORT
(oracle/ltl_oracle.c, all host threads) -> tests/golden/c2_levels.json.  The reference itself refuses this
input (1024 traces); the oracle is pinned against the reference wherever the reference runs.
Takes a few minutes of CPU.  Usage: python tests/golden/make_c2_levels.py"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import oracle_factory  # noqa: E402
from oracle import cpu_oracle  # noqa: E402
from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200.learner import learn  # noqa: E402

spec, alphabet, planted, cfg = Wl.make_config("c2_planted")
t0 = time.time()
res = learn(spec, None, alphabet, max_cost=cfg["max_cost"], core_factory=oracle_factory(cpu_oracle.max_threads()),
            budget_bytes=150 << 30)
out = {
    "generator": "tests/golden/make_c2_levels.py (CPU oracle port)", "config": {k: v for k, v in cfg.items()},
    "status": res.status, "formula": res.text, "cost": res.cost, "offered": res.stats.offered,
    "admitted": res.stats.admitted, "duplicates": res.stats.duplicates,
    "levels": [{k: v for k, v in lv.items() if k != "ms"} for lv in res.stats.levels],
    "seconds": round(time.time() - t0, 1),
}
with open(os.path.join(HERE, "c2_levels.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(out)
