# round 2: type-3 item phase breakdown (extra event codes; role 3 = softmax warp 6)
mkdir -p gpurun_out/ev3
DYLLM_NVCC_FLAGS=-DDYLLM_ATTN_EVENTS=2 python -m paper_2603_08026_b200.build --force > gpurun_out/ev3/build.log 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 4 > gpurun_out/ev3/ro.txt 2>&1; tail -60 gpurun_out/ev3/ro.txt | head -70
timeout 300 python tools/attn_events.py --mode fi --items 2 --kind 4 > gpurun_out/ev3/fi.txt 2>&1
