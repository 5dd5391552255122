#!/bin/bash
# Sort rewrite check: sort tests, then the C5 shard sweep (sort ms per eps) and
# a launch list of the S4096 sort.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "sort or pipeline or long_rows or capacity or append" > gpurun_out/sort_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sort_pytest.log
timeout 900 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S4096 > gpurun_out/sort_c5.jsonl 2>&1; echo "rc=$?" >> gpurun_out/sort_c5.jsonl
timeout 900 python scripts/c5_sweep.py --shard 0/8 --reps 1 --only S1024 >> gpurun_out/sort_c5.jsonl 2>&1; echo "rc=$?" >> gpurun_out/sort_c5.jsonl
