# round 2: FullStep GEMMs on the skinny kernel: GPU tests + default bench (with the full-recompute leg)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_d.log 2>&1
tail -1 gpurun_out/bench_d.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['clocks'], d['full_recompute'], d['roofline']['frac'], d['salient_step_roofline']['frac'], {k: v['avg_us'] for k, v in d['kernels'].items()})"
