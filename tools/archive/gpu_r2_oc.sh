# round 2: one activation chunk (R = 410, two MMAs per k-step) with stream-K splits for O / down / QKV / GU
mkdir -p gpurun_out
timeout 600 python tools/gemm_bench.py --rows 410 --one-chunk 512 --split 0,2,3,4 --reps 10 > gpurun_out/oc410.txt 2>&1; cat gpurun_out/oc410.txt
timeout 600 python tools/gemm_bench.py --rows 410 --split 0,2,4 --reps 10 --which o,down > gpurun_out/oc410b.txt 2>&1; cat gpurun_out/oc410b.txt
