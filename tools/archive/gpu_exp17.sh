mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/exp17_tests.log 2>&1; tail -3 gpurun_out/exp17_tests.log
timeout 300 python tools/gemm_bench.py --rows 205,410,1530 --split 0 --reps 10 > gpurun_out/exp17_gemm.log 2>&1
