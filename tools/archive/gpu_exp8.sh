mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp8_tests.log 2>&1; tail -3 gpurun_out/exp8_tests.log
timeout 300 python tools/gemm_bench.py --rows 15296 --reps 5 > gpurun_out/exp8_gemm.log 2>&1
timeout 300 python tools/gemm_bench.py --rows 15296 --skinny 0 --reps 5 >> gpurun_out/exp8_gemm.log 2>&1
timeout 900 python bench.py > gpurun_out/exp8_bench.log 2>&1; tail -1 gpurun_out/exp8_bench.log | cut -c1-300
