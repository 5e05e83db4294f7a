#!/bin/bash
# source-level ncu captures (SASS opcode mix) of the non-GEMM kernels of one
# config-2 step: k_crt8, k_res_cols, k_res_rows
mkdir -p gpurun_out
python tools/headline_steps.py > gpurun_out/hs_plain.log 2>&1 || { tail gpurun_out/hs_plain.log; exit 1; }
for k in k_crt8 k_res_cols k_res_rows; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k python tools/headline_steps.py > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv 2>/dev/null
  ncu -i gpurun_out/prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$k.csv 2>/dev/null
  rm -f gpurun_out/prof_$k.ncu-rep
done
ls -la gpurun_out | tail
