mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
timeout 300 python tools/select_bench.py > gpurun_out/exp54.log 2>&1
