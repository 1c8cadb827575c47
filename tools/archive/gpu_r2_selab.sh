# round 2: selection kernel 512 threads x 2 rows per warp (16 loads in flight per lane) vs 1024 x 1
mkdir -p gpurun_out
for t in 1024 512; do
  DYLLM_NVCC_FLAGS=-DDYLLM_SEL_THREADS=$t python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
  echo "threads $t"; timeout 300 python tools/select_bench.py 2>&1 | tail -4
done
python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_denoise.py -q -x > gpurun_out/pytest_sel.log 2>&1; tail -2 gpurun_out/pytest_sel.log
