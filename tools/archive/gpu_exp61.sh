mkdir -p gpurun_out
: > gpurun_out/exp61.log
for V in "def:" "norpf:-DDYLLM_FA_RPF=0" "noepit:-DDYLLM_FA_EPIT=0" "neither:-DDYLLM_FA_RPF=0 -DDYLLM_FA_EPIT=0"; do
  name=${V%%:*}; flags=${V#*:}
  rm -rf /tmp/r_$name && mkdir -p /tmp/r_$name && cp -r . /tmp/r_$name/ 2>/dev/null
  (cd /tmp/r_$name && DYLLM_NVCC_FLAGS="$flags" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1)
done
for rep in 1 2; do
for name in def norpf noepit neither; do
  (cd /tmp/r_$name && timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), d['clocks']['sm_mhz'], d['kernels']['attn']['avg_us'])") >> gpurun_out/exp61.log
done
done
