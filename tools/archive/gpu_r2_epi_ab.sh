# round 2: skinny GEMM epilogue with every row-id / residual load issued before the stores (A/B vs HEAD build)
mkdir -p gpurun_out/eab
for v in base new base new; do
  cp ab/libdyllm_$v.so paper_2603_08026_b200/libdyllm.so
  for m in ro fi; do
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_skinny --csv --log-file gpurun_out/eab/${v}_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
    python tools/ncu_summary.py launches gpurun_out/eab/${v}_$m.csv | grep gemm_skinny | sed "s/^/$v $m /"
  done
done
cp ab/libdyllm_new.so paper_2603_08026_b200/libdyllm.so
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x > gpurun_out/eab/pytest.log 2>&1; tail -2 gpurun_out/eab/pytest.log
