#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/c5_e2e.py 6.97276473038035 0/8 > gpurun_out/c5_e2e_s64.jsonl 2> gpurun_out/c5_e2e.err
