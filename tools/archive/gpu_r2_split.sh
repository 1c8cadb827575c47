# round 2: type-3 items in two stages on different warps (DYLLM_FA_SPLIT): correctness first, then A/B vs v3
mkdir -p gpurun_out/spl
cp ab/libdyllm_split.so paper_2603_08026_b200/libdyllm.so
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x > gpurun_out/spl/pytest_layer.log 2>&1; echo "layer rc=$?"; tail -2 gpurun_out/spl/pytest_layer.log
grep -E "^E " gpurun_out/spl/pytest_layer.log | head -5
timeout 600 python -m pytest tests/test_gpu_denoise.py tests/test_gpu_fullsize.py -q -x > gpurun_out/spl/pytest_more.log 2>&1; echo "more rc=$?"; tail -2 gpurun_out/spl/pytest_more.log
for v in v3 split v3 split; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:attn_fused --csv --log-file gpurun_out/spl/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/spl/${v}_$m.csv | grep attn_fused | sed "s/^/$v $m /"
  done
done
