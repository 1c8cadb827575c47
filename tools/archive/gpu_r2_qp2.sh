# round 2: qkv_post with 256 threads per row (2 rounds, all rows resident in one wave) vs 512
mkdir -p gpurun_out
for t in 512 256; do
  DYLLM_NVCC_FLAGS=-DDYLLM_QKVPOST_THREADS=$t python -m paper_2603_08026_b200.build > /dev/null 2>&1
  for m in ro fi; do
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qpt${t}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    echo "threads=$t $m: $(python tools/ncu_summary.py launches gpurun_out/qpt${t}_$m.csv | grep -E 'qkv_post')"
  done
done
python -m paper_2603_08026_b200.build > /dev/null 2>&1
