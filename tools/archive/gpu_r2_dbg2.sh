mkdir -p gpurun_out/sk
for cfg in "qkv 3" "o 3" "qkv 1" "qkv 2" "o 1" "o 2"; do
  set -- $cfg
  timeout 120 python tools/skinny_trace.py --which $1 --rows 410 --dbg $2 --per-cta > gpurun_out/sk/trd_$1_d$2.txt 2>&1
  head -12 gpurun_out/sk/trd_$1_d$2.txt
done
