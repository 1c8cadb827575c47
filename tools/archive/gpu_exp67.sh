mkdir -p gpurun_out
: > gpurun_out/exp67.log
python -m paper_2603_08026_b200.build > /dev/null 2>&1
rm -rf /tmp/r_k0 && mkdir -p /tmp/r_k0 && cp -r . /tmp/r_k0/ 2>/dev/null
(cd /tmp/r_k0 && DYLLM_NVCC_FLAGS="-DDYLLM_FA_KACT=0" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1)
for rep in 1 2; do
for name in def k0; do
  if [ $name = def ]; then D=.; else D=/tmp/r_k0; fi
  (cd $D && timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), d['clocks']['sm_mhz'], d['kernels']['attn']['avg_us'])") >> gpurun_out/exp67.log
done
done
(cd /tmp/r_k0 && timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q 2>&1 | tail -1 | sed 's/^/k0 tests: /') >> gpurun_out/exp67.log
