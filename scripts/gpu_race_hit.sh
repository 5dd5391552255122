#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/san_hit.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
os.environ["FASTED_RES_HIT"] = "2"
import paper_2508_21230_b200 as F
hd = F.to_half(F.generate_synthetic(2999, 100, seed=2999))
print(len(F.self_join(hd, 3.3)), flush=True)
PY
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 python /tmp/san_hit.py > gpurun_out/race_hit.txt 2>&1
grep -E "SUMMARY|hazard detected|Thread" gpurun_out/race_hit.txt | head -30
