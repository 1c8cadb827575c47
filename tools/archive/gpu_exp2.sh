mkdir -p gpurun_out
for w in qkv gu down; do for S in 0 64; do timeout 120 python tools/skinny_trace.py --which $w --rows 410 --split $S; done; done > gpurun_out/exp2_trace.log 2>&1
timeout 300 python tools/attn_trace.py --mode ro > gpurun_out/exp2_attn.log 2>&1
timeout 300 python tools/attn_trace.py --mode fi >> gpurun_out/exp2_attn.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/exp2_full.log 2>&1
