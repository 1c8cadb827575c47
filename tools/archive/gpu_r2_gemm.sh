# round 2: skinny GEMM chunking sweep at the RO / FI row counts + cuBLAS reference
mkdir -p gpurun_out
timeout 600 python tools/gemm_bench.py --rows 410,1530 --reps 10 > gpurun_out/gemm_auto.txt 2>&1; cat gpurun_out/gemm_auto.txt
timeout 900 python tools/gemm_bench.py --rows 410 --one-chunk 256 --chunk 256,208,176,160,144,128,112 --reps 10 > gpurun_out/gemm_chunk410.txt 2>&1; cat gpurun_out/gemm_chunk410.txt
timeout 900 python tools/gemm_bench.py --rows 1530 --chunk 256,224,208,192,176,160,144,128 --reps 10 > gpurun_out/gemm_chunk1530.txt 2>&1; cat gpurun_out/gemm_chunk1530.txt
timeout 300 python tools/cublas_ref.py > gpurun_out/cublas_ref.txt 2>&1; cat gpurun_out/cublas_ref.txt
