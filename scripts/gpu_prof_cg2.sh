#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:join_tc_kernel -s 2 -c 1 --csv --log-file gpurun_out/ncu_c4_cg2_fulllaunch.csv python scripts/ncu_join.py C4 1000064 40 > gpurun_out/ncu_c4_cg2_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_tc_kernel -s 2 -c 1 -o gpurun_out/ncu_c4_cg2 python scripts/ncu_join.py C4 131072 40 > gpurun_out/ncu_c4_cg2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy --no-symmetric --e2e-steps 1 > gpurun_out/launches_cg2.log 2>&1
