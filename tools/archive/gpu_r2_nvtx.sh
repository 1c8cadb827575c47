# round 2: GPU tests, bench, NVTX range check (kernels of one layer of a response-only step via ncu --nvtx)
mkdir -p gpurun_out/nvtx
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 1 --warmup 3 > gpurun_out/bench_nvtx.log 2>&1
tail -1 gpurun_out/bench_nvtx.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['e2e']['value'], d['clocks'], d['roofline']['frac'], {k: v['avg_us'] for k, v in d['kernels'].items()})"
timeout 600 ncu --nvtx --nvtx-include "dyllm response-only step/layer 5/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/nvtx/layer5_ro.csv python tools/profile_step.py --mode ro > gpurun_out/nvtx/log.txt 2>&1
grep -c gpu__time_duration gpurun_out/nvtx/layer5_ro.csv; tail -3 gpurun_out/nvtx/log.txt
