mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp5_tests.log 2>&1; tail -3 gpurun_out/exp5_tests.log
timeout 900 python bench.py > gpurun_out/exp5_bench.log 2>&1; tail -1 gpurun_out/exp5_bench.log | cut -c1-400
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp5_launches_ro.csv python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp5_launches_fi.csv python tools/profile_step.py --mode fi > /dev/null 2>&1
