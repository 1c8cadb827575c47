mkdir -p gpurun_out
for oc in 0 512; do timeout 300 python tools/gemm_bench.py --which o,down --rows 410 --split 0,1,2,4,8 --one-chunk $oc --reps 10; done > gpurun_out/exp25_gemm.log 2>&1
