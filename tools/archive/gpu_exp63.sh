# needs tools/_attn_head.cu = git show b51de24:paper_2603_08026_b200/csrc/attn_fused.cu (not committed)
mkdir -p gpurun_out
: > gpurun_out/exp63.log
python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1 >> gpurun_out/exp63.log
rm -rf /tmp/r_head && mkdir -p /tmp/r_head && cp -r . /tmp/r_head/ 2>/dev/null && cp tools/_attn_head.cu /tmp/r_head/paper_2603_08026_b200/csrc/attn_fused.cu
(cd /tmp/r_head && python -m paper_2603_08026_b200.build --force > /dev/null 2>&1)
rm -rf /tmp/r_t4 && mkdir -p /tmp/r_t4 && cp -r . /tmp/r_t4/ 2>/dev/null
(cd /tmp/r_t4 && DYLLM_NVCC_FLAGS="-DDYLLM_FA_T4=1" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1)
(cd /tmp/r_t4 && timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q 2>&1 | tail -1 | sed 's/^/t4 build: /') >> gpurun_out/exp63.log
for rep in 1 2; do
for name in new head; do
  if [ $name = new ]; then D=.; else D=/tmp/r_head; fi
  (cd $D && timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), d['clocks']['sm_mhz'], d['kernels']['attn']['avg_us'])") >> gpurun_out/exp63.log
done
done
