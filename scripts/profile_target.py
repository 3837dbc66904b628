#!/usr/bin/env python
"""One search of a BASELINE workload, nothing else: the command ncu wraps (see profiles/README.md).
With --stats the core times its kernels with CUDA events and the per-class totals are printed."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200.core import make_core  # noqa: E402
from paper_2402_12373_b200.learner import learn  # noqa: E402
from paper_2402_12373_b200.scheme import HashScheme  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_planted")
ap.add_argument("--max-cost", type=int, default=None)
ap.add_argument("--budget-gb", type=float, default=150.0)
ap.add_argument("--stats", action="store_true")
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--hash", default="mueller", help="fingerprint scheme (scheme.py): mueller | mueller_blocked | nh | fkp")
ap.add_argument("--unsolvable", action="store_true", help="random traces of the config's shape: every level is exhaustive")
a = ap.parse_args()
t0 = time.time()
if a.unsolvable:
    wl = dict(Wl.CONFIGS[a.config])
    spec, alphabet = Wl.random_spec(wl["n_props"], wl["n_pos"], wl["n_neg"], wl["min_len"], wl["max_len"], wl["seed"])
else:
    spec, alphabet, planted, wl = Wl.make_config(a.config)
print(f"workload {a.config}: {spec.n_pos}+{spec.n_neg} traces, max_len {spec.max_len}, generated in {time.time() - t0:.1f} s")
cores = []


def factory(*args, **kw):
    core = make_core(*args, **kw, profile=a.stats)
    real_close = core.close

    def close():
        if a.stats:
            cores.append((core.kernel_stats(), core.host_times(), core.info()))
        real_close()

    core.close = close
    return core


for rep in range(a.repeat):
    t0 = time.time()
    res = learn(spec, None, alphabet, max_cost=a.max_cost or wl["max_cost"], budget_bytes=int(a.budget_gb * (1 << 30)),
                core_factory=factory, hash=HashScheme(a.hash))
    dt = time.time() - t0
    print(f"run {rep}: {res.status} {res.text!r} cost={res.cost} offered={res.stats.offered} admitted={res.stats.admitted} "
          f"wall={dt * 1e3:.1f} ms  search={res.stats.search_seconds * 1e3:.1f} ms  "
          f"{res.stats.offered / max(res.stats.search_seconds, 1e-9) / 1e6:.1f} M cand/s  "
          f"phases {({k: round(v, 1) for k, v in res.stats.phase_ms.items()})}")
print([(lv["cost"], lv["offered"], lv["admitted"], lv.get("ms")) for lv in res.stats.levels])
if a.stats and cores:
    ks, ht, info = cores[-1]
    print(json.dumps({k: {"launches": v["launches"], "ms": round(v["ms"], 3), "GB": round(v["alg_bytes"] / 1e9, 2),
                          "alg_GBps": round(v["alg_bytes"] / 1e6 / v["ms"], 1) if v["ms"] > 0 else None}
                      for k, v in ks.items() if v["launches"]}))
    print(ht, info)
