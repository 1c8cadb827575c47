# round 2: skinny k-block width 128 vs 64 (ring depth)
mkdir -p gpurun_out/sk; timeout 300 python tools/gemm_bench.py --rows 100,205,410,1530 --kb 0,64 > gpurun_out/sk/kb.txt 2>&1; grep -v "^\s*$" gpurun_out/sk/kb.txt | tail -32
