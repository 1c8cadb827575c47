mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_skinny -s 3 -c 1 -o gpurun_out/sk_gu410 python tools/gemm_bench.py --which gu --rows 410 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_skinny -s 3 -c 1 -o gpurun_out/sk_gu1530 python tools/gemm_bench.py --which gu --rows 1530 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tcgen05 -s 3 -c 1 -o gpurun_out/std_gu1530 python tools/gemm_bench.py --which gu --rows 1530 --skinny 0 --reps 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
