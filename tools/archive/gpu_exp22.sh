mkdir -p gpurun_out
DYLLM_NVCC_FLAGS=-DDYLLM_ATTN_EVENTS=1 python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 4 > gpurun_out/exp22_ev_ro.log 2>&1
timeout 300 python tools/attn_events.py --mode full --items 1 --kind 2 > gpurun_out/exp22_ev_fi.log 2>&1
