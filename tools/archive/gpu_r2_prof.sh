# round 2: TP test rerun; ncu --set full of the selection and qkv_post kernels in a response-only step
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tp.py -q -s > gpurun_out/pytest_tp.log 2>&1; grep -E "band|passed|failed" gpurun_out/pytest_tp.log | tail -8
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"select_salient|qkv_post" -c 2 -o gpurun_out/r2_sel_qkvpost python tools/profile_step.py --mode ro > gpurun_out/ncu_selq.log 2>&1; tail -2 gpurun_out/ncu_selq.log
