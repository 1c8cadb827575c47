# round 2 final evidence after the fused a2 + a3 (FullStep + full-input steps): smoke, GPU suite, bench, reference arm, launch lists, sweeps
# launch lists of the three step kinds, sweeps (Dream, n_u, f)
mkdir -p gpurun_out/r2f4
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2f4/smoke.log 2>&1; tail -1 gpurun_out/r2f4/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2f4/pytest_gpu.log 2>&1; tail -1 gpurun_out/r2f4/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2f4/bench.json 2> gpurun_out/r2f4/bench.err; tail -1 gpurun_out/r2f4/bench.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r2f4/ref.json 2>&1; tail -1 gpurun_out/r2f4/ref.json | cut -c1-200
for m in ro fi full; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f4/launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/r2f4/launches_$m.csv > gpurun_out/r2f4/launches_$m.md; head -1 gpurun_out/r2f4/launches_$m.md
done
timeout 900 python bench.py --config dream7b --steps 1 --warmup 2 --no-cpu-baseline --full-gens 0 > gpurun_out/r2f4/dream.json 2>&1; tail -1 gpurun_out/r2f4/dream.json | cut -c1-100
for n in 2 4; do timeout 900 python bench.py --n-u $n --steps 1 --warmup 2 --no-cpu-baseline --full-gens 0 > gpurun_out/r2f4/nu$n.json 2>&1; tail -1 gpurun_out/r2f4/nu$n.json | cut -c1-100; done
for f in 0.05 0.2; do timeout 900 python bench.py --frac $f --steps 1 --warmup 2 --no-cpu-baseline --full-gens 0 > gpurun_out/r2f4/f$f.json 2>&1; tail -1 gpurun_out/r2f4/f$f.json | cut -c1-100; done
