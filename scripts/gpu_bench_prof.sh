#!/bin/bash
# Round evidence: GPU suite, bench line, ncu launch list of the bench command,
# full-launch DRAM bytes of the C4 join, ncu --set full of a C4 row slice.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy --e2e-steps 1 > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:join_tc_mc -s 1 -c 1 --csv --log-file gpurun_out/ncu_c4_full_dram.csv python scripts/ncu_join.py C4 1000064 > gpurun_out/ncu_c4_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_tc_mc -s 1 -c 1 -o gpurun_out/ncu_c4_mc_full python scripts/ncu_join.py C4 75776 > gpurun_out/ncu_c4_slice.log 2>&1
