# round 2: exact-row attention items claimed before every row-tile item: A/B (base = old order)
mkdir -p gpurun_out/xfirst
for v in base xfirst; do
  if [ $v = base ]; then F="-DDYLLM_FA_X_FIRST=0"; else F=""; fi
  DYLLM_NVCC_FLAGS="$F" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 > gpurun_out/xfirst/bench_$v.log 2>&1
  tail -1 gpurun_out/xfirst/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select')})"
  for M in ro fi; do
    if [ $M = ro ]; then R="dyllm response-only step/"; else R="dyllm full-input step/"; fi
    timeout 600 ncu --nvtx --nvtx-include "$R" -k regex:attn_fused --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max --clock-control none --csv --log-file gpurun_out/xfirst/${M}_$v.csv python tools/profile_step.py --mode $M > /dev/null 2>&1
    grep attn_fused gpurun_out/xfirst/${M}_$v.csv | grep gpu__time | awk -F'","' '{print $NF}' | tr -d '"' | awk -v m=$M '$1>20000{s+=$1;n++} END{print m, "attention main launch mean us", s/n/1000, n}'
  done
  if [ $v = xfirst ]; then timeout 900 python -m pytest tests/test_gpu_denoise.py tests/test_gpu_fullsize.py tests/test_gpu_layer.py -q -x 2>&1 | tail -2; fi
done
