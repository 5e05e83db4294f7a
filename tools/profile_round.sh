#!/bin/bash
# Round profile: launch list (all kernels of one short bench run) and one
# full ncu capture each of the mm kernel and the elementwise kernels.
# Usage (on the GPU box): bash tools/profile_round.sh <tag>
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mm_fast -c 1 -o gpurun_out/prof_mm_$TAG $CMD > gpurun_out/ncu_mm_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fast -c 8 -o gpurun_out/prof_ew_$TAG $CMD > gpurun_out/ncu_ew_$TAG.log 2>&1
ls -la gpurun_out | tail -12
