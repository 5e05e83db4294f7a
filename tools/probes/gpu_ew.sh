#!/bin/bash
# elementwise GPU check: parity tests + suite timing (+ one ncu --set full capture
# of the TMA kernel of each op named in the arguments)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_g2.py tests/test_gpu_elementwise.py -x -q > gpurun_out/ew_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ew_tests.log
tail -3 gpurun_out/ew_tests.log
timeout 300 python tools/probes/ew_time.py > gpurun_out/ew_time.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/ew_time.json'))
print(' '.join(f'{k}:{v[\"ms\"]*1000:.1f}us/{v[\"frac\"]:.2f}' for k,v in d.items()))"
for op in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tma -c 1 -o gpurun_out/prof_$op python tools/probes/ew_time.py $op > gpurun_out/ncu_$op.log 2>&1
  ncu -i gpurun_out/prof_$op.ncu-rep --page raw --csv > gpurun_out/raw_$op.csv 2>/dev/null
  ncu -i gpurun_out/prof_$op.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$op.csv 2>/dev/null
  rm -f gpurun_out/prof_$op.ncu-rep
done
