timeout 900 python -m pytest tests/test_gpu_mlp.py -q -x > gpurun_out/mlp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mlp_tests.log; tail -15 gpurun_out/mlp_tests.log
python tools/mlp_time.py 8192 2>&1 | tail -2
MCF_GEMM_F32_I8=0 python tools/mlp_time.py 8192 2>&1 | tail -2
