mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/sweep_tests.log 2>&1; tail -2 gpurun_out/sweep_tests.log
timeout 900 python bench.py --config dream7b --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_dream.json 2>&1; tail -1 gpurun_out/sweep_dream.json | cut -c1-150
for f in 0.05 0.2 0.5 1.0; do
  timeout 1200 python bench.py --frac $f --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/sweep_f$f.json 2>&1; tail -1 gpurun_out/sweep_f$f.json | cut -c1-150
done
