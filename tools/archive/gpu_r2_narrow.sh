# round 2: type-3 narrow tiles (<= 32 changed keys spread over the 4 column groups, trimmed PV): A/B
mkdir -p gpurun_out/nar
for v in base narrow; do
  if [ $v = base ]; then F="-DDYLLM_FA_NARROW=0"; else F=""; fi
  DYLLM_NVCC_FLAGS="$F" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
  for m in ro fi; do
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:attn_fused --csv --log-file gpurun_out/nar/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/nar/${v}_$m.csv | grep attn_fused | head -3
  done
  timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 > gpurun_out/nar/bench_$v.log 2>&1
  tail -1 gpurun_out/nar/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','select')})"
done
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_denoise.py tests/test_gpu_fullsize.py -q -x > gpurun_out/nar/pytest.log 2>&1; tail -3 gpurun_out/nar/pytest.log
