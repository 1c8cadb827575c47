mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -x -q > gpurun_out/exp14_tests.log 2>&1; tail -2 gpurun_out/exp14_tests.log
timeout 300 python tools/attn_events.py --mode ro --items 3 > gpurun_out/exp14_ev_ro.log 2>&1
timeout 300 python tools/attn_events.py --mode fi --items 2 > gpurun_out/exp14_ev_fi.log 2>&1
timeout 300 python tools/attn_events.py --mode full --items 2 > gpurun_out/exp14_ev_full.log 2>&1
