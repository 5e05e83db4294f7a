#!/bin/bash
# usage: bash tools/bench_sweep.sh VAR "v1 v2 ..."  -> ms_per_step per value
VAR=$1
for v in $2; do
  env $VAR=$v python bench.py --steps 5 --warmup 3 --no-extras 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', d['ms_per_step'], d['value'], d['e2e']['value'])"
done
