"""Where does learn() spend host time?  cProfile of one warm end-to-end call on the bench workload."""
import cProfile
import pstats
import sys
import time

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200.learner import learn  # noqa: E402
from paper_2402_12373_b200.traces import Specification  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_planted"
spec, al, f, cfg = Wl.make_config(name)
pc, pl = spec.chars[:spec.n_pos].copy(), spec.lengths[:spec.n_pos].copy()
nc, nl = spec.chars[spec.n_pos:].copy(), spec.lengths[spec.n_pos:].copy()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = Specification.from_arrays(pc, pl, nc, nl)
    t1 = time.perf_counter()
    r = learn(s, None, al, max_cost=cfg["max_cost"], budget_bytes=150 << 30)
    t2 = time.perf_counter()
    flush.fill_(1)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print([lv.get("ms") for lv in r.stats.levels])
    print(f"spec {1e3*(t1-t0):.2f}  learn {1e3*(t2-t1):.2f}  (search {1e3*r.stats.search_seconds:.2f})  flush {1e3*(t3-t2):.2f}")
pr = cProfile.Profile()
pr.enable()
r = learn(s, None, al, max_cost=cfg["max_cost"], budget_bytes=150 << 30)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)

# the bench's end-to-end loop: no device synchronize between calls
walls = []
for rep in range(12):
    t0 = time.perf_counter()
    s = Specification.from_arrays(pc, pl, nc, nl)
    r = learn(s, None, al, max_cost=cfg["max_cost"], budget_bytes=150 << 30)
    flush.fill_(1)
    walls.append((round(1e3 * (time.perf_counter() - t0), 2), [lv.get("ms") for lv in r.stats.levels][-4:]))
torch.cuda.synchronize()
for w in walls:
    print(w)
