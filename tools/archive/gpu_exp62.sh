mkdir -p gpurun_out
: > gpurun_out/exp62.log
for V in "a::" "b:tools/_attn_noinline.cu:" "c:tools/_attn_noinline.cu:-DDYLLM_FA_NO_T4 -DDYLLM_FA_QDEC=0"; do
  name=${V%%:*}; rest=${V#*:}; src=${rest%%:*}; flags=${rest#*:}
  rm -rf /tmp/r_$name && mkdir -p /tmp/r_$name && cp -r . /tmp/r_$name/ 2>/dev/null
  if [ -n "$src" ]; then cp $src /tmp/r_$name/paper_2603_08026_b200/csrc/attn_fused.cu; fi
  (cd /tmp/r_$name && DYLLM_NVCC_FLAGS="$flags" python -m paper_2603_08026_b200.build --force > /tmp/build_$name.log 2>&1) || echo "build $name failed" >> gpurun_out/exp62.log
done
for rep in 1 2; do
for name in a b c; do
  (cd /tmp/r_$name && timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), d['clocks']['sm_mhz'], d['kernels']['attn']['avg_us'])") >> gpurun_out/exp62.log
done
done
(cd /tmp/r_b && timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1) >> gpurun_out/exp62.log
