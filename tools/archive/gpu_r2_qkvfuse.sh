# round 2: a2 + a3 fused (EPI_QKV): correctness, then launch lists and bench vs v3
mkdir -p gpurun_out/qf
cp ab/libdyllm_qf.so paper_2603_08026_b200/libdyllm.so
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_denoise.py tests/test_gpu_tp.py tests/test_gpu_fp32.py -q -x > gpurun_out/qf/pytest1.log 2>&1; echo "tests1 rc=$?"; tail -1 gpurun_out/qf/pytest1.log; grep -E "^E " gpurun_out/qf/pytest1.log | head -5
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_kernels.py tests/test_gpu_batch.py -q -x > gpurun_out/qf/pytest2.log 2>&1; echo "tests2 rc=$?"; tail -1 gpurun_out/qf/pytest2.log; grep -E "^E " gpurun_out/qf/pytest2.log | head -5
for v in v3 qf v3 qf; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qf/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/qf/${v}_$m.csv | sed -n '1p;5,12p' | grep -E "launches|gemm_skinny_kernel<0|gemm_skinny_kernel<4|qkv_post|gather_rmsnorm" | sed "s/^/$v $m /"
  done
done
cp ab/libdyllm_qf.so paper_2603_08026_b200/libdyllm.so
timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 > gpurun_out/qf/bench_qf.log 2>&1; tail -1 gpurun_out/qf/bench_qf.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"value\"],1), d[\"clocks\"][\"sm_mhz\"], d[\"full_recompute\"][\"tokens_per_s\"])"
