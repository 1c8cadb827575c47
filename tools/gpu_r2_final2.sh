# round 2 (resumed session) final evidence: ncu --set full of the dominant kernel class (gate/up skinny
# GEMM, layer 5 of a response-only and a full-input step) and of the attention main launch (layer 5),
# the new every-sequence full-size parity test
mkdir -p gpurun_out/f2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k every_sequence > gpurun_out/f2/pytest_every.log 2>&1; tail -2 gpurun_out/f2/pytest_every.log
for m in ro fi; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_skinny -s 22 -c 1 -o gpurun_out/f2/gu_$m python tools/profile_step.py --mode $m > gpurun_out/f2/ncu_gu_$m.log 2>&1; tail -1 gpurun_out/f2/ncu_gu_$m.log
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -s 10 -c 1 -o gpurun_out/f2/attn_$m python tools/profile_step.py --mode $m > gpurun_out/f2/ncu_attn_$m.log 2>&1; tail -1 gpurun_out/f2/ncu_attn_$m.log
done
for r in gu_ro gu_fi attn_ro attn_fi; do python tools/ncu_summary.py report gpurun_out/f2/$r.ncu-rep > gpurun_out/f2/$r.md 2>&1; head -4 gpurun_out/f2/$r.md | tail -1; done
