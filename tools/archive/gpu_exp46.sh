mkdir -p gpurun_out
DYLLM_NVCC_FLAGS="-DDYLLM_ATTN_EVENTS=1" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 3 --kind 2 > gpurun_out/exp46.log 2>&1
