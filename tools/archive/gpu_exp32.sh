mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py --rows 1530,1600 --reps 10 > gpurun_out/exp32_gemm.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/exp32_tests.log 2>&1; tail -1 gpurun_out/exp32_tests.log
