mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:select_salient -c 1 -o gpurun_out/r1e_select python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -c 1 -o gpurun_out/r1e_attn python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_skinny -s 3 -c 1 -o gpurun_out/r1e_skinny_gu python tools/profile_step.py --mode ro > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
