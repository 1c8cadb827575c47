# round 2 (resumed session): sanitizer pass over the changed skinny epilogue / qkv_post (denoise tests, small configs)
mkdir -p gpurun_out/san3
K="test_denoise_tiny or test_denoise_small128_gqa"
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_denoise.py -q -x -k "$K" > gpurun_out/san3/${tool}_denoise.log 2>&1; echo "$tool rc=$?"; tail -1 gpurun_out/san3/${tool}_denoise.log
done
