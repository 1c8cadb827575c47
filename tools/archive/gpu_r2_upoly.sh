# round 2: FMA-pipe exps for every other key of U tiles after the first (full-input prompt tiles): A/B
mkdir -p gpurun_out/upoly
for v in upoly base; do
  if [ $v = upoly ]; then F="-DDYLLM_FA_UPOLY=1"; else F=""; fi
  DYLLM_NVCC_FLAGS="$F" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 > gpurun_out/upoly/bench_$v.log 2>&1
  tail -1 gpurun_out/upoly/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select')})"
  timeout 600 ncu --nvtx --nvtx-include "dyllm full-input step/" -k regex:attn_fused --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/upoly/fi_$v.csv python tools/profile_step.py --mode fi > /dev/null 2>&1
  grep attn_fused gpurun_out/upoly/fi_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | awk '$1>20000{s+=$1;n++} END{print "FI attention main launch mean us", s/n/1000, n}'
  if [ $v = upoly ]; then timeout 900 python -m pytest tests/test_gpu_denoise.py tests/test_gpu_fullsize.py tests/test_gpu_layer.py -q -x 2>&1 | tail -2; fi
done
