mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py --which qkv,gu --rows 410 --split 0,2,4,8,32 --reps 10 > gpurun_out/exp34.log 2>&1
timeout 300 python tools/gemm_bench.py --which qkv,gu --rows 410 --split 0,2,4,8 --one-chunk 512 --reps 10 >> gpurun_out/exp34.log 2>&1
