mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/exp53.log 2>&1; tail -3 gpurun_out/exp53.log
