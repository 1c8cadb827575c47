mkdir -p gpurun_out
python -m paper_2603_08026_b200.build --force > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r1l_smoke.log 2>&1; tail -1 gpurun_out/r1l_smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r1l_tests.log 2>&1; tail -1 gpurun_out/r1l_tests.log
timeout 900 python bench.py > gpurun_out/r1l_bench.json 2>gpurun_out/r1l_bench.err; tail -1 gpurun_out/r1l_bench.json | cut -c1-200
for m in ro fi; do timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1l_launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; done
