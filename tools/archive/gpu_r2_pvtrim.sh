# round 2: type-3 P.dV issued over ceil(nkP / 16) k-steps only (no other change): tests, then A/B
mkdir -p gpurun_out/pvt
cp ab/libdyllm_pvt.so paper_2603_08026_b200/libdyllm.so
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_denoise.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pvt/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pvt/pytest.log
for v in base pvt base pvt; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:attn_fused --csv --log-file gpurun_out/pvt/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/pvt/${v}_$m.csv | grep attn_fused | sed "s/^/$v $m /"
  done
done
cp ab/libdyllm_pvt.so paper_2603_08026_b200/libdyllm.so
