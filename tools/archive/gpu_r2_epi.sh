# round 2: skinny epilogue decomposition (no loads / MMAs; then no stores, no transpose)
for W in qkv o; do for D in 3 7 11 15; do
  echo "$W dbg=$D $(timeout 120 python tools/skinny_trace.py --which $W --rows 410 --dbg $D | grep -E 'tfull0|published|epi_done' | tr -s ' ' | tr '\n' ' ')"
done; done
for D in 0 4 8; do timeout 120 python tools/gemm_bench.py --rows 410 --dbg $D --which qkv,o,gu,down | grep -v "^\s*$"; done
