# round 2: BASELINE configs C3 (Dream-7B), C4 (salient-fraction sweep incl. 100%), C5 per-GPU shards
# (batch 32 / 64 on one GPU), f2 (n_u = 2, 4): one timed generation each, no full-recompute leg
mkdir -p gpurun_out/r2sw
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 1 --warmup 2 --full-gens 0 "$@" > gpurun_out/r2sw/$name.log 2>&1
  tail -1 gpurun_out/r2sw/$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), d['clocks']['sm_mhz'], d['roofline']['frac'], d['salient_step_roofline']['frac'], d['salient_fraction']['f_run'])" 2>/dev/null || tail -3 gpurun_out/r2sw/$name.log; }
for f in 0.05 0.2 0.5 1.0; do run frac$f --frac $f; done
run dream --config dream7b
run nu2 --n-u 2
run nu4 --n-u 4
run batch32 --batch 32
run batch64 --batch 64
