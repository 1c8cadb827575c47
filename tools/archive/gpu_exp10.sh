mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q > gpurun_out/exp10_tests.log 2>&1; tail -2 gpurun_out/exp10_tests.log
timeout 300 python tools/attn_trace.py --mode ro > gpurun_out/exp10_attn.log 2>&1
timeout 300 python tools/attn_trace.py --mode fi >> gpurun_out/exp10_attn.log 2>&1
timeout 300 python tools/attn_trace.py --mode full >> gpurun_out/exp10_attn.log 2>&1
