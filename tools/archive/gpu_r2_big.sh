# round 2: FullStep-size GEMMs: skinny (device M) vs the standard kernel (host M, bench) vs cuBLAS
mkdir -p gpurun_out
timeout 600 python tools/gemm_bench.py --rows 15296 --reps 5 > gpurun_out/gemm_15296.txt 2>&1; cat gpurun_out/gemm_15296.txt
