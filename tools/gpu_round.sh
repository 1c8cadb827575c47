mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -2 gpurun_out/bench.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c_launches_ro.csv python tools/profile_step.py --mode ro > gpurun_out/ncu_ro.log 2>&1; tail -2 gpurun_out/ncu_ro.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c_launches_fi.csv python tools/profile_step.py --mode fi > gpurun_out/ncu_fi.log 2>&1; tail -2 gpurun_out/ncu_fi.log
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -c 1 -o gpurun_out/r1c_attn_fused python tools/profile_step.py --mode ro > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
