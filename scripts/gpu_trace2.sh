#!/bin/bash
# Who sees tfull late (NOEPI, suspend vs spin waits), and the sort launch list at C5 S4096.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/trace_res.py C3 75776 256,8448,0,8192 > gpurun_out/trace2.txt 2>&1
AB_SHARD=0/8 timeout 600 python scripts/ab_env.py C3 6 "X=0" "F=8192" "F=256" "F=8448" > gpurun_out/spin_ab.txt 2>&1
bash scripts/gpu_sort_prof.sh
timeout 900 python -m pytest tests/test_cli.py tests/test_dist_gpu.py -m gpu -q > gpurun_out/r2c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_pytest.log
