# round 2: qkv_post launch bounds A/B (launch lists), skinny GEMM at FullStep row counts
mkdir -p gpurun_out
for lb in 2 1; do
  DYLLM_NVCC_FLAGS=-DDYLLM_QKVPOST_LB=$lb python -m paper_2603_08026_b200.build > /dev/null 2>&1
  for m in ro fi; do
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qp${lb}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    echo "lb=$lb $m: $(python tools/ncu_summary.py launches gpurun_out/qp${lb}_$m.csv | grep -E 'qkv_post|select')"
  done
done
python -m paper_2603_08026_b200.build > /dev/null 2>&1
timeout 600 python tools/gemm_bench.py --rows 15296 --reps 5 > gpurun_out/gemm_15296.txt 2>&1; cat gpurun_out/gemm_15296.txt
