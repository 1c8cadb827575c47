mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -c 1 -o gpurun_out/r1i_attn_fi python tools/profile_step.py --mode fi > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -c 1 -o gpurun_out/r1i_attn_ro python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:select_salient -c 1 -o gpurun_out/r1i_select_fi python tools/profile_step.py --mode fi > /dev/null 2>&1
ls gpurun_out/r1i*
