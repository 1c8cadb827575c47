mkdir -p gpurun_out
DYLLM_NVCC_FLAGS="-DDYLLM_ATTN_EVENTS=1 -DFA_EXP_NOSTORE" python -m paper_2603_08026_b200.build --force > gpurun_out/exp42.log 2>&1
timeout 300 python tools/attn_events.py --mode fi --items 3 > gpurun_out/exp42_fi.log 2>&1
