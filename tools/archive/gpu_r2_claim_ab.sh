# round 2: attention producer claims two items ahead: A/B vs v3
mkdir -p gpurun_out/aab
for v in v3 v4 v3 v4; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:attn_fused --csv --log-file gpurun_out/aab/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/aab/${v}_$m.csv | grep attn_fused | sed "s/^/$v $m /"
  done
done
cp ab/libdyllm_v4.so paper_2603_08026_b200/libdyllm.so
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_denoise.py tests/test_gpu_fullsize.py tests/test_gpu_batch.py -q -x > gpurun_out/aab/pytest.log 2>&1; tail -2 gpurun_out/aab/pytest.log
timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 > gpurun_out/aab/bench_v4.log 2>&1; tail -1 gpurun_out/aab/bench_v4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn','o_gemm','down_gemm','qkv_post')})"
