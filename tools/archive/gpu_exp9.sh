mkdir -p gpurun_out
timeout 300 python tools/attn_trace.py --mode ro > gpurun_out/exp9_attn.log 2>&1
timeout 300 python tools/attn_trace.py --mode fi >> gpurun_out/exp9_attn.log 2>&1
