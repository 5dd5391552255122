#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "sharding" > gpurun_out/pytest_shard.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_shard.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_tc_res -s 1 -c 1 -o gpurun_out/ncu_c3_now python scripts/ncu_join.py C3 75776 > gpurun_out/ncu_c3_now.log 2>&1
