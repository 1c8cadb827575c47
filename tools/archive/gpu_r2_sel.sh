# round 2: TP tests + per-sequence threshold in the selection kernel: full GPU suite + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tp.py -q -s > gpurun_out/pytest_tp.log 2>&1; grep -E "band|passed|failed" gpurun_out/pytest_tp.log | tail -8
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 > gpurun_out/bench_sel.log 2>&1
tail -1 gpurun_out/bench_sel.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select','qkv_post','o_gemm')})"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_ro.csv python tools/profile_step.py --mode ro > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/r2s_launches_ro.csv | head -12
