#!/bin/bash
# Per-config kernel throughput (tune.py: CUDA-event time per launch, clocks, power).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest_cfg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_cfg.log
timeout 600 python scripts/tune.py C2 20 "CG=0" > gpurun_out/tune_cfg_c2.log 2>&1
timeout 900 python scripts/tune.py C3 5 "CG=0" > gpurun_out/tune_cfg_c3.log 2>&1
timeout 900 python scripts/tune.py C4 3 "CG=0" > gpurun_out/tune_cfg_c4.log 2>&1
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 1 > gpurun_out/c5_cfg.jsonl 2> gpurun_out/c5_cfg.err
