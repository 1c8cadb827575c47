# round 2: fused similarity partials (f3) + parallel build_u: GPU tests, same-box A/B, launch lists
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -8 gpurun_out/pytest_gpu.log
for o in 1 0; do
  timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 --lib-opt 9=$o > gpurun_out/bench_cos$o.log 2>&1
  tail -1 gpurun_out/bench_cos$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cos=$o', d['value'], d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select','qkv_post')})"
done
for m in ro fi; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches_$m.csv python tools/profile_step.py --mode $m > gpurun_out/ncu_$m.log 2>&1; tail -1 gpurun_out/ncu_$m.log
done
