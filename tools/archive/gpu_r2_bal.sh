# round 2: per-kernel SM busy-time balance (sm__cycles_active avg / max) over one response-only and one full-input step
mkdir -p gpurun_out/bal
for M in ro fi; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_elapsed.avg --clock-control none --csv --log-file gpurun_out/bal/$M.csv python tools/profile_step.py --mode $M > /dev/null 2>&1
done
ls -la gpurun_out/bal
