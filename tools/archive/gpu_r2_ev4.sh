# round 2: type-3 phase breakdown with the narrow tiles (events build)
mkdir -p gpurun_out/ev4
DYLLM_NVCC_FLAGS=-DDYLLM_ATTN_EVENTS=2 python -m paper_2603_08026_b200.build --force > gpurun_out/ev4/build.log 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 4 > gpurun_out/ev4/ro.txt 2>&1; grep -v "^      " gpurun_out/ev4/ro.txt | head -120
