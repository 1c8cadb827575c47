# round 2: k-block-granular stream-K (split = k-blocks per tile) at M = 410 / 1530
mkdir -p gpurun_out/sk
timeout 300 python tools/gemm_bench.py --rows 410,1530 --split 0,8,16,32 --which qkv,o,down > gpurun_out/sk/kg.txt 2>&1; grep -v "^\s*$" gpurun_out/sk/kg.txt | tail -24
timeout 300 python tools/gemm_bench.py --rows 410 --split 0,8,16,32 --one-chunk 512 --which qkv,gu > gpurun_out/sk/kg_oc.txt 2>&1; grep -v "^\s*$" gpurun_out/sk/kg_oc.txt | tail -8
for cfg in "qkv 32 0" "gu 32 512" "o 32 0" "down 96 0"; do
  set -- $cfg
  timeout 120 python tools/skinny_trace.py --which $1 --rows 410 --split $2 --one-chunk $3 --per-cta > gpurun_out/sk/tr_$1_s$2_c$3.txt 2>&1
  head -12 gpurun_out/sk/tr_$1_s$2_c$3.txt
done
