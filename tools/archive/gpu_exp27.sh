mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_unmask.py -x -q > gpurun_out/exp27_tests.log 2>&1; tail -15 gpurun_out/exp27_tests.log
