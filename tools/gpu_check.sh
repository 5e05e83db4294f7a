#!/bin/bash
# quick GPU check: linalg/ozaki/mlp tests + bench headline + e2e (+ optional extra command)
python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_linalg.py tests/test_gpu_mlp.py -x -q > gpurun_out/t.log 2>&1
tail -2 gpurun_out/t.log
python bench.py --steps 5 --warmup 3 --no-extras 2>/dev/null | tail -1 > gpurun_out/bench_oz.json
python -c "
import json; d=json.load(open('gpurun_out/bench_oz.json')); r=d['roofline']
print('step', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value'], 'phases', r.get('step_phases_ms'), 'fallback', r.get('fallback_outputs'), 'frac', r['frac'])"
