# round 2: spill-free default attention + f3 variant tests + bench + GEMM chunk sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 > gpurun_out/bench_c.log 2>&1
tail -1 gpurun_out/bench_c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items()})"
bash tools/gpu_r2_gemm.sh
