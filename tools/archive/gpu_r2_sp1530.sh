# round 2: stream-K split granularities at the full-input row count (M = 1530)
mkdir -p gpurun_out
timeout 900 python tools/gemm_bench.py --rows 1530 --split 0,2,3,4,8 --reps 10 > gpurun_out/sp1530.txt 2>&1; cat gpurun_out/sp1530.txt
