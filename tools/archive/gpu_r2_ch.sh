# round 2: activation chunks of up to 512 rows (two MMAs per k-step) for M > 512
mkdir -p gpurun_out/sk
timeout 600 python tools/gemm_bench.py --rows 600,1024,1530,2048,4096,15296 --chunk 0,320,384,448,512 --reps 10 > gpurun_out/sk/ch.txt 2>&1; grep -v "^\s*$" gpurun_out/sk/ch.txt | tail -120
