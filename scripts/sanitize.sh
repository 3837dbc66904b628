#!/bin/bash
# compute-sanitizer evidence (race / memory checks of the dedup and compaction kernels), run under gpurun:
#   scripts/sanitize.sh <tag>
# memcheck (global / shared out-of-bounds, misaligned), racecheck (shared-memory hazards: the cp.async.bulk / mbarrier
# ring of k_screen, the block scans of k_scan) and synccheck (barrier misuse) over (1) smoke(), (2) a row-split run with
# multi-word rows, the fused NOT and a budget cut, (3) the device-resident specification kernels.
# Outputs: gpurun_out/<tag>_sanitize_<tool>_<case>.log (tails are kept under profiles/).
tag=${1:-r02}
cat > /tmp/sanitize_case.py <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
case = sys.argv[1]
if case == "smoke":
    import __graft_entry__ as g
    g.smoke()
elif case == "rowsplit":
    # many rows x few candidates (row split + k_finalize), 3 words per row, solver cut, then a budget cut
    from paper_2402_12373_b200 import workloads as Wl
    from paper_2402_12373_b200.learner import learn
    spec, alphabet = Wl.random_spec(2, 300, 300, 70, 150, 5)
    r = learn(spec, None, alphabet, max_cost=5)
    print("rowsplit", r.status, (r.text or "")[:60], r.stats.offered)
    spec, alphabet = Wl.random_spec(3, 260, 260, 20, 64, 9)
    r = learn(spec, None, alphabet, max_cost=5, budget_bytes=3000 * (520 * 8 + 16))
    print("budget", r.status, r.stats.offered, r.stats.admitted)
    spec, alphabet = Wl.random_spec(3, 2100, 2100, 5, 32, 11)     # half-width store, fused NOT levels
    r = learn(spec, None, alphabet, max_cost=5)
    print("halfwidth", r.status, r.stats.offered, r.stats.admitted)
elif case == "traces":
    from paper_2402_12373_b200 import learner
    from paper_2402_12373_b200.learner import learn
    learner.DEVICE_SPEC_MIN_CHARS = 0
    rng = np.random.default_rng(3)
    R, L = 5000, 40
    lengths = rng.integers(20, L + 1, size=R).astype(np.int64)  # long enough for 5000 random traces to be distinct
    chars = rng.integers(0, 8, size=(R, L)).astype(np.uint16)
    r = learn((chars[:2500], lengths[:2500]), (chars[2500:], lengths[2500:]), 3, max_cost=4)
    print("traces", r.status, r.stats.offered, r.stats.h2d_bytes)
PY
for tool in memcheck racecheck synccheck; do
  for case in smoke rowsplit traces; do
    out=gpurun_out/${tag}_sanitize_${tool}_${case}.log
    echo "== $tool $case"; date
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python /tmp/sanitize_case.py $case > $out 2>&1
    echo "exit $?" >> $out
    tail -4 $out
  done
done
