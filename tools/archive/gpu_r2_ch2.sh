# round 2: one-round chunking for O / down at M > 512 (auto) vs 256-row chunks (C = 256)
mkdir -p gpurun_out/sk
timeout 600 python tools/gemm_bench.py --rows 600,800,1024,1300,1530,1800,2048 --chunk 0,256 --which o,down,qkv,gu --reps 20 > gpurun_out/sk/ch2.txt 2>&1; tail -3 gpurun_out/sk/ch2.txt
