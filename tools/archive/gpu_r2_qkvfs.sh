# round 2: a2 + a3 fused in FullSteps only (DYLLM_OPT_QKV_FUSED default 1): full GPU suite, FullStep launch list, bench
mkdir -p gpurun_out/qfs
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/qfs/pytest_gpu.log 2>&1; tail -1 gpurun_out/qfs/pytest_gpu.log; grep -E "^FAILED" gpurun_out/qfs/pytest_gpu.log | head
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qfs/full.csv python tools/profile_step.py --mode full > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/qfs/full.csv | head -12
timeout 800 python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/qfs/bench.json 2>&1; tail -1 gpurun_out/qfs/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'], d['full_recompute']['tokens_per_s'], {k: v['avg_us'] for k, v in d['kernels'].items() if 'full' in k})"
