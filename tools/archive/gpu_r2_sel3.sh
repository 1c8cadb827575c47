# round 2: selection kernel in two shapes (256 threads x 4 CTAs/SM for full-input launches)
mkdir -p gpurun_out
timeout 300 python tools/select_trace.py 2>&1 | tail -2
timeout 300 python tools/select_bench.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_denoise.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_sel3.log 2>&1; tail -2 gpurun_out/pytest_sel3.log
