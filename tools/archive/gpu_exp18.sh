mkdir -p gpurun_out
for oc in 512 256; do timeout 300 python tools/gemm_bench.py --rows 300,410,512 --one-chunk $oc --reps 10; done > gpurun_out/exp18_gemm.log 2>&1
