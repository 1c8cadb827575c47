# round 2: CTA-wide radix select in the selection kernel: trace + tests + bench
mkdir -p gpurun_out
timeout 300 python tools/select_trace.py 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 > gpurun_out/bench_sel2.log 2>&1
tail -1 gpurun_out/bench_sel2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select')})"
