#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest_dyn.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dyn.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:join_tc_mc -s 1 -c 1 --csv --log-file gpurun_out/dram_c5_dyn.csv python scripts/ncu_join.py C5 75776 0 7.2300123612099165 > gpurun_out/dram_c5_dyn.log 2>&1
timeout 900 python scripts/tune.py C4 2 "CG=0" "CG=0,DYN=0" > gpurun_out/tune_c4_dyn.log 2>&1
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S > gpurun_out/c5_dyn.jsonl 2> gpurun_out/c5_dyn.err
