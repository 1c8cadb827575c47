# round 2: skinny GEMM decomposition: no operand loads (dbg 1) / no MMAs (dbg 2), clocks sampled
mkdir -p gpurun_out/sk
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 250 > gpurun_out/sk/clk_dbg.csv &
SMI=$!
for D in 0 1 2 3; do
  timeout 300 python tools/gemm_bench.py --rows 410,1530 --dbg $D --reps 50 > gpurun_out/sk/dbg$D.txt 2>&1; echo "dbg $D"; grep -v "^\s*$" gpurun_out/sk/dbg$D.txt | tail -8
  timeout 300 python tools/gemm_bench.py --rows 410 --split 32 --which qkv --dbg $D --reps 50 | tail -1
done
kill $SMI
awk -F, 'NR>1{print $2, $3, $4}' gpurun_out/sk/clk_dbg.csv | sort | uniq -c | sort -rn | head -12
