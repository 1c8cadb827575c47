mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r1h_bench.json 2>gpurun_out/r1h_bench.err; tail -1 gpurun_out/r1h_bench.json | cut -c1-150
for m in ro fi full; do timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1h_launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; done
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -c 1 -o gpurun_out/r1h_attn_ro python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_skinny -s 2 -c 1 -o gpurun_out/r1h_skinny_gu_ro python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:select_salient -c 1 -o gpurun_out/r1h_select_ro python tools/profile_step.py --mode ro > /dev/null 2>&1
ls gpurun_out/r1h*
