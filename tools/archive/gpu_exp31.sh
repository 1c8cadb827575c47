mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x > gpurun_out/exp31_tests.log 2>&1; tail -2 gpurun_out/exp31_tests.log
for m in ro fi; do timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp31_launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; done
