mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > gpurun_out/exp45.log 2>&1
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x >> gpurun_out/exp45.log 2>&1; tail -3 gpurun_out/exp45.log
for T in 32 0 32 0; do
echo "T4=$T" >> gpurun_out/exp45.log
timeout 300 python tools/step_gap.py --mode ro --opt 7=$T 2>&1 | head -1 >> gpurun_out/exp45.log
done
timeout 300 python tools/step_gap.py --mode fi --opt 7=32 2>&1 | head -1 >> gpurun_out/exp45.log
