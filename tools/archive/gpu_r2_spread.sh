# round 2: exact-row queries spread over the four TMEM lane quadrants (qx_spread): tests, then A/B vs v3
mkdir -p gpurun_out/sp
cp ab/libdyllm_spread.so paper_2603_08026_b200/libdyllm.so
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_denoise.py tests/test_gpu_tp.py -q -x > gpurun_out/sp/pytest1.log 2>&1; echo "tests1 rc=$?"; tail -1 gpurun_out/sp/pytest1.log; grep -E "^E |^FAILED" gpurun_out/sp/pytest1.log | head -5
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_batch.py tests/test_gpu_analysis.py -q -x > gpurun_out/sp/pytest2.log 2>&1; echo "tests2 rc=$?"; tail -1 gpurun_out/sp/pytest2.log; grep -E "^E |^FAILED" gpurun_out/sp/pytest2.log | head -5
for v in v3 spread v3 spread; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sp/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/sp/${v}_$m.csv | sed -n '1p;5,9p' | grep -E "launches|attn_fused" | sed "s/^/$v $m /"
  done
done
cp ab/libdyllm_spread.so paper_2603_08026_b200/libdyllm.so
