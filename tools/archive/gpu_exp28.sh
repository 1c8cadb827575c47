mkdir -p gpurun_out
DYLLM_NVCC_FLAGS="-DDYLLM_ATTN_EVENTS=1" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode full --items 1 --kind 2 > gpurun_out/exp28_ev_a.log 2>&1
DYLLM_NVCC_FLAGS="-DDYLLM_ATTN_EVENTS=1 -DFA_NO_VOTE=1" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode full --items 1 --kind 2 > gpurun_out/exp28_ev_b.log 2>&1
