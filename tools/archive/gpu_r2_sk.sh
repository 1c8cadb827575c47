# round 2: skinny GEMM phase traces of split configurations at M = 410 (why split-K loses)
set -x
mkdir -p gpurun_out/sk
for cfg in "qkv 0 0" "qkv 2 0" "qkv 3 0" "gu 0 0" "gu 0 512" "gu 2 512" "down 0 0" "o 0 0"; do
  set -- $cfg
  timeout 120 python tools/skinny_trace.py --which $1 --rows 410 --split $2 --one-chunk $3 --per-cta > gpurun_out/sk/tr_$1_s$2_c$3.txt 2>&1
  head -14 gpurun_out/sk/tr_$1_s$2_c$3.txt
done
timeout 300 python tools/gemm_bench.py --rows 410 --split 0,2,3,4 --one-chunk 512 --which qkv,gu,down > gpurun_out/sk/oc512.txt 2>&1; cat gpurun_out/sk/oc512.txt | grep -v "^\s*$" | tail -14
