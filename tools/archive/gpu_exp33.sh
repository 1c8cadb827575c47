mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py --rows 205,410,1530 --reps 10 > gpurun_out/exp33_a.log 2>&1
DYLLM_NVCC_FLAGS="-DSK_NO_TMA=1" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/gemm_bench.py --rows 205,410,1530 --reps 10 > gpurun_out/exp33_b.log 2>&1
