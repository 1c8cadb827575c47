mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > gpurun_out/final_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final_smoke.log 2>&1; tail -2 gpurun_out/final_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; tail -2 gpurun_out/final_tests.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2>gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-160
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/final_ref.json 2>&1; tail -1 gpurun_out/final_ref.json | cut -c1-200
timeout 900 python bench.py --config dream7b --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/final_dream.json 2>&1; tail -1 gpurun_out/final_dream.json | cut -c1-120
for f in 0.05 0.2 0.5; do timeout 1200 python bench.py --frac $f --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final_f$f.json 2>&1; tail -1 gpurun_out/final_f$f.json | cut -c1-120; done
timeout 900 python bench.py --n-u 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final_nu2.json 2>&1; tail -1 gpurun_out/final_nu2.json | cut -c1-120
timeout 900 python bench.py --n-u 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final_nu4.json 2>&1; tail -1 gpurun_out/final_nu4.json | cut -c1-120
