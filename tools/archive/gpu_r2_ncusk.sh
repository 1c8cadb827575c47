# round 2: ncu --set full of the skinny QKV GEMM at M = 410 (normal and loads-only)
mkdir -p gpurun_out/ncusk
for D in 0 2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny --launch-skip 3 --launch-count 1 \
  -o gpurun_out/ncusk/qkv410_d$D -f python tools/gemm_bench.py --rows 410 --which qkv --reps 2 --dbg $D > gpurun_out/ncusk/log_d$D.txt 2>&1
tail -2 gpurun_out/ncusk/log_d$D.txt
done
ls -la gpurun_out/ncusk
