mkdir -p gpurun_out
timeout 300 python tools/attn_events.py --mode ro --items 3 > gpurun_out/exp13_ev_ro.log 2>&1
timeout 300 python tools/attn_events.py --mode fi --items 2 > gpurun_out/exp13_ev_fi.log 2>&1
