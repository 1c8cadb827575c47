# round 2 (resumed session): full GPU tests, smoke, launch list of a response-only step, default bench
mkdir -p gpurun_out/res
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/res/pytest_gpu.log 2>&1; tail -3 gpurun_out/res/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/res/smoke.log 2>&1; tail -1 gpurun_out/res/smoke.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/res/launches_ro.csv python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/res/launches_fi.csv python tools/profile_step.py --mode fi > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/res/launches_ro.csv | head -14
python tools/ncu_summary.py launches gpurun_out/res/launches_fi.csv | head -14
timeout 900 python bench.py > gpurun_out/res/bench.log 2>&1; tail -c 600 gpurun_out/res/bench.log
