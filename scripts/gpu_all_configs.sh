#!/bin/bash
# Per-config kernel throughput with the product's kernel choice (tune.py passes the
# kernel-form hints the engine sets from the expected output, engine.form_hints).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/tune.py C2 20 "CG=0" "CG=0" > gpurun_out/tune_cfg_c2.log 2>&1
timeout 900 python scripts/tune.py C3 5 "CG=0" "CG=0" > gpurun_out/tune_cfg_c3.log 2>&1
timeout 900 python scripts/tune.py C4 3 "CG=0" "CG=0" > gpurun_out/tune_cfg_c4.log 2>&1
timeout 1500 python scripts/c5_sweep.py --shard 0/8 --reps 2 > gpurun_out/c5_cfg.jsonl 2> gpurun_out/c5_cfg.err
