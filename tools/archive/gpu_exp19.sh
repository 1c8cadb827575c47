mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp19_tests.log 2>&1; tail -2 gpurun_out/exp19_tests.log
timeout 900 python bench.py > gpurun_out/exp19_bench.log 2>&1; tail -1 gpurun_out/exp19_bench.log | cut -c1-200
for m in ro fi full; do timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp19_launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; done
