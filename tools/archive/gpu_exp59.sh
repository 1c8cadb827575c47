mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
: > gpurun_out/exp59.log
for T in 32 0 32 0; do
  timeout 900 python bench.py --no-cpu-baseline --lib-opt 7=$T 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('T4=$T', round(d['value'],1), d['clocks']['sm_mhz'], d['kernels']['attn']['avg_us'])" >> gpurun_out/exp59.log
done
