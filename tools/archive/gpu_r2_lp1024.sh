# round 2: the paper's representative prompt length L_P = 1024 at C2, f = 0.1 (and 0.05)
mkdir -p gpurun_out/lp
timeout 900 python bench.py --no-cpu-baseline --lp 1024 --steps 1 --warmup 3 > gpurun_out/lp/lp1024_f0.1.log 2>&1; tail -c 300 gpurun_out/lp/lp1024_f0.1.log
timeout 900 python bench.py --no-cpu-baseline --lp 1024 --frac 0.05 --steps 1 --warmup 3 --full-gens 0 > gpurun_out/lp/lp1024_f0.05.log 2>&1; tail -c 300 gpurun_out/lp/lp1024_f0.05.log
