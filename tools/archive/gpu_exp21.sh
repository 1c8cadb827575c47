mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q > gpurun_out/exp21_tests.log 2>&1; tail -3 gpurun_out/exp21_tests.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp21_alltests.log 2>&1; tail -3 gpurun_out/exp21_alltests.log
timeout 900 python bench.py > gpurun_out/exp21_bench.log 2>&1; tail -1 gpurun_out/exp21_bench.log | cut -c1-200
for m in ro fi; do timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp21_launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; done
