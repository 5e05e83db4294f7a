#!/bin/bash
# Round profile: launch list (all kernels of one short bench run) and one
# full ncu capture each of the mm kernel, the elementwise kernels and the
# MLP step kernels.  Usage (on the GPU box): bash tools/profile_round.sh <tag>
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "bench failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mm_fast -c 1 -o gpurun_out/prof_mm_$TAG $CMD > gpurun_out/ncu_mm_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tma|k_fast" -c 12 -o gpurun_out/prof_ew_$TAG $CMD > gpurun_out/ncu_ew_$TAG.log 2>&1
MLP="python tools/mlp_time.py 8192"
$MLP > gpurun_out/plain_mlp_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mm_fast|k_gemm|k_bias_act|k_ce|k_rowsum|k_sgd" -c 12 -o gpurun_out/prof_mlp_$TAG $MLP > gpurun_out/ncu_mlp_$TAG.log 2>&1
ls -la gpurun_out | tail -14
# summaries on the box (the .ncu-rep files together exceed gpurun's 64 MiB pull limit)
python tools/ncu_summary.py gpurun_out/launches_$TAG.csv gpurun_out/prof_mm_$TAG.ncu-rep gpurun_out/prof_ew_$TAG.ncu-rep > gpurun_out/summary_$TAG.md 2>&1
python tools/ncu_summary.py gpurun_out/launches_$TAG.csv gpurun_out/prof_mlp_$TAG.ncu-rep > gpurun_out/summary_mlp_$TAG.md 2>&1
for r in mm ew mlp; do ncu -i gpurun_out/prof_${r}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${r}_$TAG.csv 2>/dev/null; done
ncu -i gpurun_out/prof_mm_$TAG.ncu-rep --page source --csv > gpurun_out/source_mm_$TAG.csv 2>/dev/null
rm -f gpurun_out/prof_ew_$TAG.ncu-rep gpurun_out/prof_mlp_$TAG.ncu-rep
