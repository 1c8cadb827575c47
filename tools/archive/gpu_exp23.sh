mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp23_tests.log 2>&1; tail -2 gpurun_out/exp23_tests.log
timeout 900 python bench.py > gpurun_out/exp23_bench.log 2>&1; tail -1 gpurun_out/exp23_bench.log | cut -c1-200
