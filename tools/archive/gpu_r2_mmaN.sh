# round 2: skinny main-loop time vs activation rows with no operand loads (MMA issue cost vs N)
for M in 64 128 192 240 256 288 320 384 410 416 448 512; do
  echo "M=$M $(timeout 120 python tools/skinny_trace.py --which qkv --rows $M --dbg 1 --one-chunk 512 | grep -E 'mma_done')"
done
for M in 128 256 410 512; do
  echo "loads M=$M $(timeout 120 python tools/skinny_trace.py --which qkv --rows $M --dbg 2 --one-chunk 512 | grep -E 'prod_done')"
  echo "both  M=$M $(timeout 120 python tools/skinny_trace.py --which qkv --rows $M --dbg 0 --one-chunk 512 | grep -E 'mma_done')"
done
