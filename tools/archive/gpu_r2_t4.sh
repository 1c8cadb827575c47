# round 2: transposed exact-row tiles (type 4) compiled in: event timeline + same-box bench A/B
mkdir -p gpurun_out
for v in t4 base; do
  if [ $v = t4 ]; then F="-DDYLLM_FA_T4=1"; else F=""; fi
  DYLLM_NVCC_FLAGS="$F" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 > gpurun_out/bench_$v.log 2>&1
  tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['clocks']['sm_mhz'], {k: v['avg_us'] for k, v in d['kernels'].items() if k in ('attn',)})"
done
DYLLM_NVCC_FLAGS="-DDYLLM_FA_T4=1 -DDYLLM_ATTN_EVENTS=1" python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
timeout 300 python tools/attn_events.py --mode ro --items 4 > gpurun_out/attn_events_ro_t4.txt 2>&1; head -20 gpurun_out/attn_events_ro_t4.txt
python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
