# round 2: ncu --set full of the selection kernel and the O-proj / FFN-down skinny GEMM with the final kernels (layer 5)
mkdir -p gpurun_out/sf
for m in ro fi; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:select_salient -s 5 -c 1 -o gpurun_out/sf/sel_$m python tools/profile_step.py --mode $m > /dev/null 2>&1
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_skinny -s 21 -c 1 -o gpurun_out/sf/o_$m python tools/profile_step.py --mode $m > /dev/null 2>&1
done
for r in sel_ro sel_fi o_ro o_fi; do python tools/ncu_summary.py report gpurun_out/sf/$r.ncu-rep > gpurun_out/sf/$r.md 2>&1; sed -n 4p gpurun_out/sf/$r.md; done
