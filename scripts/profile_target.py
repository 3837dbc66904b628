#!/usr/bin/env python
"""One search of a BASELINE workload, nothing else: the command ncu wraps (see profiles/README.md)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200.learner import learn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_planted")
ap.add_argument("--max-cost", type=int, default=None)
ap.add_argument("--budget-gb", type=float, default=150.0)
a = ap.parse_args()
spec, alphabet, planted, wl = Wl.make_config(a.config)
res = learn(spec, None, alphabet, max_cost=a.max_cost or wl["max_cost"], budget_bytes=int(a.budget_gb * (1 << 30)))
print(res.status, res.text, res.cost, res.stats.offered, res.stats.admitted)
print([(lv["cost"], lv["offered"], lv["admitted"], lv.get("ms")) for lv in res.stats.levels])
