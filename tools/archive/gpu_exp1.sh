mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py --rows 205,410 --split 0,1,2,3,4,8,16,64 --reps 10 > gpurun_out/exp1_gemm.log 2>&1
timeout 300 python tools/gemm_bench.py --rows 1530 --skinny 0 --reps 10 >> gpurun_out/exp1_gemm.log 2>&1
timeout 300 python tools/attn_trace.py --mode ro > gpurun_out/exp1_attn.log 2>&1
timeout 300 python tools/attn_trace.py --mode fi >> gpurun_out/exp1_attn.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/exp1_full.log 2>&1
