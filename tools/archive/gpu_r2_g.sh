# round 2: empty fixup launches leave before setup; qkv_post 256 threads: tests, launch list, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_ro.csv python tools/profile_step.py --mode ro > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/g_ro.csv | head -14
timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 > gpurun_out/bench_g.log 2>&1
tail -1 gpurun_out/bench_g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select','qkv_post')})"
