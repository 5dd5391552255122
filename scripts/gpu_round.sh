#!/bin/bash
cd "$(dirname "$0")/.."
bash scripts/gpu_final.sh
bash scripts/gpu_all_configs.sh
