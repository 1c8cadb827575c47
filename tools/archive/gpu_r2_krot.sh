# round 2: skinny GEMM k-block rotation per weight block (activation reads of concurrent pairs staggered)
mkdir -p gpurun_out/sk
timeout 400 python tools/gemm_bench.py --rows 410,1530 --krot 0,1,7,13 > gpurun_out/sk/krot.txt 2>&1; grep -v "^\s*$" gpurun_out/sk/krot.txt | tail -32
timeout 300 python tools/gemm_bench.py --rows 410 --split 32 --krot 0,7 --which qkv,o,down > gpurun_out/sk/krot_s32.txt 2>&1; grep -v "^\s*$" gpurun_out/sk/krot_s32.txt | tail -6
