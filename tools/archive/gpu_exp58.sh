mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
# RO step, layer 10: skinny launches in order qkv(<0>), o(<1>), gu(<2>), down(<1>) per layer
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_skinny -s 40 -c 4 -o gpurun_out/r1l_skinny_ro python tools/profile_step.py --mode ro > /dev/null 2>&1
ls -la gpurun_out/r1l_skinny_ro.ncu-rep
