mkdir -p gpurun_out
DYLLM_NVCC_FLAGS="-DDYLLM_ATTN_EVENTS=1 -DFA_EXP_NOSTORE" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 4 --kind 3 > gpurun_out/exp39_k3.log 2>&1
DYLLM_NVCC_FLAGS="-DFA_EXP_NOSTORE" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/step_gap.py --mode ro > gpurun_out/exp39.log 2>&1
