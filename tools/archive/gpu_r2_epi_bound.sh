# round 2: in-step upper bound of the skinny GEMM epilogue's store / transpose cost (dbg hooks skip them)
mkdir -p gpurun_out/eb
for o in none 12=4 12=12 none; do
  if [ $o = none ]; then L=""; else L="--lib-opt $o"; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 $L > gpurun_out/eb/b_$o.log 2>&1
  tail -1 gpurun_out/eb/b_$o.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if 'gemm' in k and 'full' not in k and 'lm' not in k})"
done
