# round 2: fp32-parity mode tests + compute-sanitizer passes on the small configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x > gpurun_out/fp32.log 2>&1; tail -15 gpurun_out/fp32.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_denoise.py -q -x -k "test_denoise_tiny or test_denoise_small128_gqa" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -6 gpurun_out/sanitizer_$tool.log
done
