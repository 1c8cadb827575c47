mkdir -p gpurun_out
: > gpurun_out/exp47.log
for PF in 1 0 1 0; do
DYLLM_NVCC_FLAGS="-DDYLLM_FA_PF=$PF" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
echo "PF=$PF" >> gpurun_out/exp47.log
timeout 300 python tools/step_gap.py --mode ro 2>&1 | head -1 >> gpurun_out/exp47.log
timeout 300 python tools/step_gap.py --mode fi 2>&1 | head -1 >> gpurun_out/exp47.log
done
python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 >> gpurun_out/exp47.log
