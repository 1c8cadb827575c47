# needs tools/_attn_kernels_head.cu = git show HEAD:paper_2603_08026_b200/csrc/kernels.cu (not committed)
mkdir -p gpurun_out
: > gpurun_out/exp64.log
python -m paper_2603_08026_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1 >> gpurun_out/exp64.log
rm -rf /tmp/r_head && mkdir -p /tmp/r_head && cp -r . /tmp/r_head/ 2>/dev/null && cp tools/_attn_kernels_head.cu /tmp/r_head/paper_2603_08026_b200/csrc/kernels.cu
(cd /tmp/r_head && python -m paper_2603_08026_b200.build --force > /dev/null 2>&1)
for rep in 1 2; do
for name in new head; do
  if [ $name = new ]; then D=.; else D=/tmp/r_head; fi
  (cd $D && timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), d['clocks']['sm_mhz'], d['kernels']['select']['avg_us'], d['kernels']['attn']['avg_us'])") >> gpurun_out/exp64.log
done
done
