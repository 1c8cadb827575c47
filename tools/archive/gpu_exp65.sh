mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
for m in ro fi; do timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1m_launches_$m.csv python tools/profile_step.py --mode $m > /dev/null 2>&1; done
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -s 20 -c 1 -o gpurun_out/r1m_attn_ro python tools/profile_step.py --mode ro > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:attn_fused -s 20 -c 1 -o gpurun_out/r1m_attn_fi python tools/profile_step.py --mode fi > /dev/null 2>&1
ls gpurun_out/r1m*
