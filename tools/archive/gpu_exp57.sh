mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -s 20 -c 1 -o gpurun_out/r1l_attn_ro python tools/profile_step.py --mode ro > /dev/null 2>&1
ls -la gpurun_out/r1l_attn_ro.ncu-rep
