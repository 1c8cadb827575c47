# round 2: calibrated fixed-tau C2 run (the paper's rule), natural tau 0.99, f4 analysis, analysis test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_analysis.py -q -x > gpurun_out/pytest_analysis.log 2>&1; tail -3 gpurun_out/pytest_analysis.log
timeout 900 python bench.py --select-mode tau --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 > gpurun_out/bench_tau.log 2>&1; tail -c 1200 gpurun_out/bench_tau.log
timeout 900 python bench.py --select-mode tau --tau 0.99 --no-cpu-baseline --steps 1 --warmup 3 --full-gens 0 > gpurun_out/bench_tau099.log 2>&1; tail -c 800 gpurun_out/bench_tau099.log
timeout 600 python tools/paper_analysis.py --out gpurun_out/paper_analysis_llada8b.json > gpurun_out/paper_analysis.txt 2>&1; tail -30 gpurun_out/paper_analysis.txt
