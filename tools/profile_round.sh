#!/bin/bash
# Round profile: launch list (all kernels of one short bench run) and full ncu
# captures of the tensor-core mm kernels (one int8 GEMM, the digit, combine
# and fallback kernels), the elementwise kernels and the MLP step kernels.
# Summaries are written on the box (the .ncu-rep files exceed gpurun's pull
# limit).  Usage (on the GPU box): bash tools/profile_round.sh <tag>
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "bench failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cutlass -s 8 -c 1 -o gpurun_out/prof_gemm_$TAG $CMD > gpurun_out/ncu_gemm_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_slice|k_combine|k_fallback|k_rowexp|k_colmax" -c 6 -o gpurun_out/prof_oz_$TAG $CMD > gpurun_out/ncu_oz_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tma|k_fast" -c 8 -o gpurun_out/prof_ew_$TAG $CMD > gpurun_out/ncu_ew_$TAG.log 2>&1
# the headline step alone (kernel shares of one step)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/step_launches_$TAG.csv python tools/headline_steps.py > /dev/null 2>&1
python tools/step_shares.py gpurun_out/step_launches_$TAG.csv > gpurun_out/step_shares_$TAG.md 2>&1
MLP="python tools/mlp_time.py 8192"
$MLP > gpurun_out/plain_mlp_$TAG.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_gemm|k_bias_act|k_ce|k_rowsum|k_sgd" -c 10 -o gpurun_out/prof_mlp_$TAG $MLP > gpurun_out/ncu_mlp_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_$TAG.csv gpurun_out/prof_gemm_$TAG.ncu-rep gpurun_out/prof_oz_$TAG.ncu-rep gpurun_out/prof_ew_$TAG.ncu-rep > gpurun_out/summary_$TAG.md 2>&1
python tools/ncu_summary.py gpurun_out/launches_$TAG.csv gpurun_out/prof_mlp_$TAG.ncu-rep > gpurun_out/summary_mlp_$TAG.md 2>&1
for r in gemm oz ew mlp; do ncu -i gpurun_out/prof_${r}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${r}_$TAG.csv 2>/dev/null; done
rm -f gpurun_out/prof_ew_$TAG.ncu-rep gpurun_out/prof_mlp_$TAG.ncu-rep gpurun_out/prof_oz_$TAG.ncu-rep
ls -la gpurun_out | tail -20
