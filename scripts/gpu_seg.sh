#!/bin/bash
# Segmented upload + APPEND: tests, the segment-launch kernel form, bench e2e.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/seg.txt
: > $out
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "append or segmented or pipeline or resident" >> $out 2>&1
python scripts/seg_forms.py >> $out 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-accuracy --no-symmetric --e2e-steps 5 > gpurun_out/bench_seg.json 2> gpurun_out/bench_seg.err
python3 -c "
import json
d=json.loads(open('gpurun_out/bench_seg.json').read().strip().split(chr(10))[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'e2e s/step', d['e2e']['seconds_per_step'], 'clocks', d['clocks'])
for p in d['e2e']['phases_per_step']:
    e=p['engine'][0]; print(' wall', p['wall_s'], 'h2d', p['h2d_s'], 'kern', p['join_kernels_s'], 'tail', p['sort_d2h_not_hidden_s'], 'timeline', e['host_ms'].get('gpu_timeline', [])[:3])
" >> $out 2>&1
tail -5 gpurun_out/bench_seg.err >> $out
cat $out
