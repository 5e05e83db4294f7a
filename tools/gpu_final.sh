#!/bin/bash
# end-of-round capture: GPU tests, default bench (both arms), smoke, the headline
# step's ncu launch list and the MLP step's
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/step_launches.csv python tools/headline_steps.py > /dev/null 2>&1
python tools/step_shares.py gpurun_out/step_launches.csv > gpurun_out/step_shares.md 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/mlp_step_launches.csv python tools/probes/mlp_steps.py > /dev/null 2>&1
python tools/step_shares.py gpurun_out/mlp_step_launches.csv > gpurun_out/mlp_step_shares.md 2>&1
head -14 gpurun_out/step_shares.md
# launch list of the bench command itself (short, headline + config 0 only)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/bench_under_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/bench_launches.csv > gpurun_out/bench_launches.md 2>&1
head -30 gpurun_out/bench_launches.md
