# round 2: skinny ring stages sized to the activation rows: GEMM tests + chunk sweep + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_kernels.log 2>&1; tail -3 gpurun_out/pytest_kernels.log
timeout 900 python tools/gemm_bench.py --rows 410 --one-chunk 256 --chunk 256,208,160,128,96 --reps 10 > gpurun_out/ring410.txt 2>&1; cat gpurun_out/ring410.txt
timeout 900 python tools/gemm_bench.py --rows 410,1530 --reps 10 > gpurun_out/ring_auto.txt 2>&1; cat gpurun_out/ring_auto.txt
timeout 900 python tools/gemm_bench.py --rows 1530 --chunk 256,208,192,160,128 --reps 10 > gpurun_out/ring1530.txt 2>&1; cat gpurun_out/ring1530.txt
