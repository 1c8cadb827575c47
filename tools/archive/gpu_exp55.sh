mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > gpurun_out/exp55.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x >> gpurun_out/exp55.log 2>&1; tail -3 gpurun_out/exp55.log
timeout 300 python tools/select_bench.py >> gpurun_out/exp55.log 2>&1
timeout 300 python tools/step_gap.py --mode ro 2>&1 | head -1 >> gpurun_out/exp55.log
timeout 300 python tools/step_gap.py --mode fi 2>&1 | head -1 >> gpurun_out/exp55.log
