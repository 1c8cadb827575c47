mkdir -p gpurun_out
DYLLM_NVCC_FLAGS="-DDYLLM_FA_2ISSUE=0" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
sed -n '/^timeout 120/,/^echo/p' tools/gpu_exp51.sh > /tmp/run51.sh
bash /tmp/run51.sh; tail -3 gpurun_out/exp51.log
timeout 300 python tools/step_gap.py --mode ro 2>&1 | head -1 >> gpurun_out/exp51.log
timeout 300 python tools/step_gap.py --mode fi 2>&1 | head -1 >> gpurun_out/exp51.log
