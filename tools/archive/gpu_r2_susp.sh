# round 2: mbarrier waits with a suspend-time hint (waiting warps stop spinning) vs v3: whole-step launch lists A/B/A/B
mkdir -p gpurun_out/sus
cp ab/libdyllm_susp.so paper_2603_08026_b200/libdyllm.so
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -q -x > gpurun_out/sus/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/sus/pytest.log
for v in v3 susp v3 susp; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sus/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/sus/${v}_$m.csv | sed -n '1p;5,9p' | sed "s/^/$v $m /"
  done
done
