# round 2: compute-sanitizer after the barrier fix: synccheck / memcheck on denoise, fp32, TP tests
mkdir -p gpurun_out/san
K="test_denoise_tiny or test_denoise_small128_gqa"
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_denoise.py -q -x -k "$K" > gpurun_out/san/synccheck_denoise.log 2>&1; echo "synccheck denoise rc=$?"; tail -3 gpurun_out/san/synccheck_denoise.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_tp.py tests/test_gpu_fp32.py -q -x -k "tiny or full_step or nccl" > gpurun_out/san/memcheck_tp_fp32.log 2>&1; echo "memcheck tp/fp32 rc=$?"; tail -3 gpurun_out/san/memcheck_tp_fp32.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_tp.py -q -x -k "full_step" > gpurun_out/san/synccheck_tp.log 2>&1; echo "synccheck tp rc=$?"; tail -3 gpurun_out/san/synccheck_tp.log
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_denoise.py -q -x -k "test_denoise_tiny" > gpurun_out/san/initcheck_denoise.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/san/initcheck_denoise.log
