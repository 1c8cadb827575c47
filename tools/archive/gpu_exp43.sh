mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > gpurun_out/exp43.log 2>&1
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x >> gpurun_out/exp43.log 2>&1; tail -2 gpurun_out/exp43.log
timeout 300 python tools/step_gap.py --mode ro >> gpurun_out/exp43.log 2>&1
timeout 300 python tools/step_gap.py --mode fi >> gpurun_out/exp43.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -s 20 -c 1 -o gpurun_out/r1l_attn_fi python tools/profile_step.py --mode fi > /dev/null 2>&1
