# round 2: tensor-parallel loopback group on one GPU + full GPU suite + step gap
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tp.py -q -x > gpurun_out/pytest_tp.log 2>&1; tail -30 gpurun_out/pytest_tp.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -6 gpurun_out/pytest_gpu.log
timeout 300 python tools/step_gap.py --mode ro > gpurun_out/step_gap_ro.txt 2>&1; tail -5 gpurun_out/step_gap_ro.txt
timeout 300 python tools/step_gap.py --mode fi > gpurun_out/step_gap_fi.txt 2>&1; tail -5 gpurun_out/step_gap_fi.txt
