#!/bin/bash
# New GPU tests (CLI accuracy/bench, two-process shards), the augment
# attribution A/B at C3, and the Fig. 8 (|D|, d) sweep through `fasted bench`.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py tests/test_dist_gpu.py -m gpu -q -x > gpurun_out/r2b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest.log
bash scripts/gpu_aug.sh
timeout 1500 python -m paper_2508_21230_b200.cli bench --ns 1000,2154,4641,10000,21544,46416,100000,215443,464159,1000000 --dims 64,128,256,512,1024,2048,4096 --repeats 3 --csv gpurun_out/sweep_fig8.csv --manifest gpurun_out/sweep_fig8.json > gpurun_out/sweep_fig8.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_fig8.log
