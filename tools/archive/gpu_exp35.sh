mkdir -p gpurun_out
timeout 300 python tools/step_gap.py --mode ro > gpurun_out/exp35.log 2>&1
timeout 300 python tools/step_gap.py --mode fi >> gpurun_out/exp35.log 2>&1
