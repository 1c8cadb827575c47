# round 2: FI attention with / without incremental prompt statistics (same box), launch lists, events
mkdir -p gpurun_out
for o in 1 0; do
  timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 --lib-opt 8=$o > gpurun_out/bench_pinc$o.log 2>&1
  tail -1 gpurun_out/bench_pinc$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pinc=$o', d['value'], d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select')})"
done
for m in ro fi; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_launches_$m.csv python tools/profile_step.py --mode $m > gpurun_out/ncu_$m.log 2>&1; tail -1 gpurun_out/ncu_$m.log
done
DYLLM_NVCC_FLAGS=-DDYLLM_ATTN_EVENTS=1 python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode fi > gpurun_out/attn_events_fi.txt 2>&1; head -40 gpurun_out/attn_events_fi.txt
python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
