# round 2: D22 (mask token never committed): full GPU suite, smoke, batch-64 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 --batch 64 > gpurun_out/b64.log 2>&1
tail -1 gpurun_out/b64.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch64', round(d['value'],1), d['clocks']['sm_mhz'], d['roofline']['frac'], d['salient_step_roofline']['frac'])" || tail -3 gpurun_out/b64.log
