# round 2 final evidence: edited GPU tests, launch lists of the three step kinds, ncu --set full of the
# attention kernel (response-only and full-input launches), default bench line (with cpu_baseline)
mkdir -p gpurun_out/r2f
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_tp.py -q > gpurun_out/r2f/pytest_edited.log 2>&1; tail -4 gpurun_out/r2f/pytest_edited.log
for m in ro fi full; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f/launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
done
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -c 1 -o gpurun_out/r2f/attn_ro python tools/profile_step.py --mode ro > gpurun_out/r2f/ncu_attn_ro.log 2>&1; tail -1 gpurun_out/r2f/ncu_attn_ro.log
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -c 1 -o gpurun_out/r2f/attn_fi python tools/profile_step.py --mode fi > gpurun_out/r2f/ncu_attn_fi.log 2>&1; tail -1 gpurun_out/r2f/ncu_attn_fi.log
timeout 900 python bench.py > gpurun_out/r2f/bench.log 2>&1; tail -c 400 gpurun_out/r2f/bench.log
