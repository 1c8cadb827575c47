# round 2: qkv_post with the epoch tag read up front and rewritten after the row (no load behind a barrier): A/B vs v2
mkdir -p gpurun_out/qab
for v in v2 v3 v2 v3; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:qkv_post --csv --log-file gpurun_out/qab/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/qab/${v}_$m.csv | grep qkv_post | sed "s/^/$v $m /"
  done
done
cp ab/libdyllm_v3.so paper_2603_08026_b200/libdyllm.so
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_denoise.py tests/test_gpu_fullsize.py -q -x > gpurun_out/qab/pytest.log 2>&1; tail -2 gpurun_out/qab/pytest.log
