"""Where do small searches spend their time?  (BASELINE config 1 runs 9 cost levels of a few hundred candidates each.)
Prints, per search: wall, time inside the library's run_level calls, the library's own device-wait time, kernel
launches; then a cProfile of one call.   python scripts/small_level_probe.py [config] [reps] [name=value ...]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_12373_b200 import workloads as Wl  # noqa: E402
from paper_2402_12373_b200 import core as C  # noqa: E402
from paper_2402_12373_b200.learner import learn  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1_tiny"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
opts = dict(kv.split("=") for kv in sys.argv[3:])
if "native_loop" in opts:  # 0: one run_level call per cost level from learner.py instead of ltl_core_run_search
    from paper_2402_12373_b200 import learner as _L

    _L.Enumeration.native_loop = bool(int(opts.pop("native_loop")))
spec, al, f, cfg = Wl.make_config(name)
P = (spec.chars[: spec.n_pos].copy(), spec.lengths[: spec.n_pos].copy())
N = (spec.chars[spec.n_pos:].copy(), spec.lengths[spec.n_pos:].copy())

acc = {"run_level": 0.0, "calls": 0, "sync": 0.0, "launches": 0}
real_run_level = C.CudaCore.run_level
real_run_search = C.CudaCore.run_search
real_close = C.CudaCore.close


def timed_run_level(self, segs):
    t0 = time.perf_counter()
    out = real_run_level(self, segs)
    acc["run_level"] += time.perf_counter() - t0
    acc["calls"] += 1
    return out


def timed_run_search(self, *a, **kw):
    t0 = time.perf_counter()
    out = real_run_search(self, *a, **kw)
    acc["run_level"] += time.perf_counter() - t0
    acc["calls"] += len(out[5])
    return out


def close(self):
    if getattr(self, "_h", None):
        acc["sync"] += self.host_times()["sync_ms"]
        acc["launches"] += sum(v["launches"] for v in self.kernel_stats().values())
    real_close(self)


C.CudaCore.run_level = timed_run_level
C.CudaCore.run_search = timed_run_search
C.CudaCore.close = close
C.CudaCore.__del__ = close


def factory(*a, **kw):
    core = C.make_core(*a, **kw)
    for k, v in opts.items():
        core.set_option(k, int(v))
    return core


def once(arrays):
    if arrays:
        return learn(P, N, al, max_cost=cfg["max_cost"])
    return learn(spec, None, al, max_cost=cfg["max_cost"], core_factory=factory if opts else None)


for arrays in (False, True):
    for _ in range(20):
        r = once(arrays)
    for k in acc:
        acc[k] = 0
    t0 = time.perf_counter()
    for _ in range(reps):
        r = once(arrays)
    wall = (time.perf_counter() - t0) / reps
    print(f"{name} {'array pairs (device-resident spec)' if arrays else 'Specification (host-packed)'}: "
          f"{1e3 * wall:.3f} ms per learn(); in run_level {1e3 * acc['run_level'] / reps:.3f} ms over {acc['calls'] // reps} levels; "
          f"library device-wait {acc['sync'] / reps:.3f} ms; kernel launches {acc['launches'] // reps}; "
          f"search {1e3 * r.stats.search_seconds:.3f} ms; phases {({k: round(v, 3) for k, v in r.stats.phase_ms.items()})}")
    print("   levels ms:", [lv.get("ms") for lv in r.stats.levels])
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    once(False)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
