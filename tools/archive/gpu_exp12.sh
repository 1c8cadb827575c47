mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp12_tests.log 2>&1; tail -2 gpurun_out/exp12_tests.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp12_launches_ro.csv python tools/profile_step.py --mode ro > /dev/null 2>&1
