mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/exp3_full.log 2>&1
