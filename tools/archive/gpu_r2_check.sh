# round 2 (resumed session): full GPU suite, smoke, default bench with the committed kernels
mkdir -p gpurun_out/chk
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/chk/pytest_gpu.log 2>&1; tail -3 gpurun_out/chk/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/chk/smoke.log 2>&1; tail -1 gpurun_out/chk/smoke.log
timeout 900 python bench.py > gpurun_out/chk/bench.log 2>&1; tail -1 gpurun_out/chk/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['clocks'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'])"
