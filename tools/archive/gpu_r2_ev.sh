# round 2: attention event timelines (response-only and full-input launches)
mkdir -p gpurun_out
DYLLM_NVCC_FLAGS=-DDYLLM_ATTN_EVENTS=1 python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 4 > gpurun_out/attn_events_ro.txt 2>&1; head -32 gpurun_out/attn_events_ro.txt
timeout 300 python tools/attn_events.py --mode fi --items 2 > gpurun_out/attn_events_fi.txt 2>&1; head -26 gpurun_out/attn_events_fi.txt
python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
