#!/bin/bash
# Final evidence run of a round on the GPU box: the full GPU test suite, smoke(), the default bench line (all shapes) and
# the reference arm, the per-shape ncu launch lists + full captures, the sanitizer runs.  Outputs in gpurun_out/<tag>_*.
tag=${1:-r02f}
timeout 1900 python -m pytest tests -m gpu -x -q --timeout 400 2>&1 | tail -6 > gpurun_out/${tag}_gputests.log; cat gpurun_out/${tag}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err; tail -c 300 gpurun_out/${tag}_bench_default.json; echo
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> /dev/null; tail -c 400 gpurun_out/${tag}_bench_reference.json; echo
bash scripts/gpu_profile_configs.sh $tag c1_tiny c2_planted c3_long c4_many c5_deep 2>&1 | grep -E "^==|bench:|total" | cut -c1-200 | tail -30
# (compute-sanitizer is closed on this pool since job r02g: scripts/sanitize.sh is run by hand where it is open)
