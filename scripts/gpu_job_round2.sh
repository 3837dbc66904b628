set -x
timeout 1500 python -m pytest tests/test_gpu_traces.py tests/test_reference_driven.py tests/test_sharded_gpu.py -m gpu -x -q --timeout 400 2>&1 | tail -15 > gpurun_out/s6_tests.log; cat gpurun_out/s6_tests.log
for b in 4 8 32 64; do LTL_CORE_OPTIONS=order_block_bytes=$((b<<20)) timeout 300 python bench.py --config c2_planted --configs none --steps 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('c2 block MB $b', round(d['value']/1e6,3), round(d['ms_per_step'],2), d['roofline']['kernel_ms_by_class']['materialize'])"; done
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/s6_launches_c2.csv python scripts/profile_target.py --config c2_planted > gpurun_out/s6_launches_c2.log 2>&1; tail -2 gpurun_out/s6_launches_c2.log
LTL_CORE_OPTIONS=order_mat=0 timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/s6_launches_c2_noorder.csv python scripts/profile_target.py --config c2_planted > gpurun_out/s6_launches_c2_noorder.log 2>&1
bash scripts/sanitize.sh r02 2>&1 | tail -40
timeout 600 python scripts/soak.py --seconds 240 --seed 11 2>&1 | tail -5 > gpurun_out/s6_soak.log; cat gpurun_out/s6_soak.log
