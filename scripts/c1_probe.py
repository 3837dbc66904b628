#!/usr/bin/env python
"""Where a small search spends its time: N searches of a BASELINE shape, wall time per phase of Enumeration.run() and the
kernel classes.  `python scripts/c1_probe.py [config] [n] [LTL_CORE_OPTIONS]`"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1_tiny"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if len(sys.argv) > 3:
    os.environ["LTL_CORE_OPTIONS"] = sys.argv[3]
import torch  # noqa: E402

from paper_2402_12373_b200 import learner as L  # noqa: E402
from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200.core import CudaCore  # noqa: E402

spec, alphabet, _planted, wl = Wl.make_config(cfg)
mc = wl["max_cost"]
real = CudaCore.run_search
acc = {"run_search": 0.0, "learn": 0.0}


def timed(self, *a, **kw):
    t = time.perf_counter()
    out = real(self, *a, **kw)
    acc["run_search"] += time.perf_counter() - t
    return out


CudaCore.run_search = timed
for k in range(n + 5):
    if k == 5:
        acc = {"run_search": 0.0, "learn": 0.0}
        torch.cuda.synchronize()
    t = time.perf_counter()
    r = L.learn(spec, None, alphabet, max_cost=mc)
    acc["learn"] += time.perf_counter() - t
print(cfg, os.environ.get("LTL_CORE_OPTIONS", ""), r.status, r.text, "per search: learn %.3f ms, run_search %.3f ms" % (1e3 * acc["learn"] / n, 1e3 * acc["run_search"] / n),
      [(x["cost"], x["offered"], x.get("ms")) for x in r.stats.levels])
