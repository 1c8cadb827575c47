# round 2: synccheck / initcheck after non-aligned named barriers and defined list buffers; tests; bench
mkdir -p gpurun_out/san
K="test_denoise_tiny or test_denoise_small128_gqa"
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_denoise.py -q -x -k "$K" > gpurun_out/san/synccheck_denoise.log 2>&1; echo "synccheck denoise rc=$?"; tail -2 gpurun_out/san/synccheck_denoise.log
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_denoise.py -q -x -k "test_denoise_tiny" > gpurun_out/san/initcheck_denoise.log 2>&1; echo "initcheck rc=$?"; tail -2 gpurun_out/san/initcheck_denoise.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_denoise.py -q -x -k "$K" > gpurun_out/san/memcheck_denoise.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/san/memcheck_denoise.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 > gpurun_out/bench_h.log 2>&1
tail -1 gpurun_out/bench_h.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select')})"
bash tools/gpu_r2_sp1530.sh
