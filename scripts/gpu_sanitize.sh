#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/san.py <<'PY'
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2508_21230_b200 as F
for n, d, eps in ((2000, 200, 5.4), (1500, 520, 8.6), (3000, 64, 2.6)):
    hd = F.to_half(F.generate_synthetic(n, d, seed=n))
    a = F.self_join(hd, eps); b = F.self_join(hd, eps, symmetric=True)
    c = F.self_join(hd, eps, mode="exact")
    print(n, d, len(a), len(b), len(c), flush=True)
PY
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
