mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
for w in o down qkv gu; do timeout 120 python tools/skinny_trace.py --which $w --rows 410; done > gpurun_out/exp40.log 2>&1
for w in o down; do timeout 120 python tools/skinny_trace.py --which $w --rows 1550; done >> gpurun_out/exp40.log 2>&1
