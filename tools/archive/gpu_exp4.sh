mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/exp4_tests.log 2>&1; tail -3 gpurun_out/exp4_tests.log
timeout 300 python tools/gemm_bench.py --rows 205,410 --split 0,1,2,4,64 --reps 10 > gpurun_out/exp4_gemm.log 2>&1
for w in qkv gu; do for S in 0 64; do timeout 120 python tools/skinny_trace.py --which $w --rows 410 --split $S; done; done > gpurun_out/exp4_trace.log 2>&1
