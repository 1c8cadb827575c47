mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > gpurun_out/exp38.log 2>&1
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x >> gpurun_out/exp38.log 2>&1; tail -2 gpurun_out/exp38.log
timeout 300 python tools/step_gap.py --mode ro >> gpurun_out/exp38.log 2>&1
timeout 300 python tools/step_gap.py --mode fi >> gpurun_out/exp38.log 2>&1
DYLLM_NVCC_FLAGS=-DDYLLM_ATTN_EVENTS=1 python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 4 --kind 3 > gpurun_out/exp38_k3.log 2>&1
