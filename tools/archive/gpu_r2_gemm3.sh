# round 2: ncu --set full with source of the QKV / O skinny GEMM at M = 410; cuBLAS kernel configs
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_skinny -c 1 -o gpurun_out/r2_skinny_qkv410 python tools/gemm_bench.py --which qkv --rows 410 --reps 2 > gpurun_out/ncu_sk1.log 2>&1; tail -2 gpurun_out/ncu_sk1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_skinny -c 1 -o gpurun_out/r2_skinny_o410 python tools/gemm_bench.py --which o --rows 410 --reps 2 > gpurun_out/ncu_sk2.log 2>&1; tail -2 gpurun_out/ncu_sk2.log
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__registers_per_thread,launch__shared_mem_per_block_dynamic --csv python tools/cublas_ref.py > gpurun_out/cublas_cfg.csv 2>&1
grep -v "^==" gpurun_out/cublas_cfg.csv | python -c "
import csv,sys,collections
rows=list(csv.DictReader(sys.stdin))
d=collections.OrderedDict()
for r in rows: d.setdefault((r['ID'], r['Kernel Name'][:100]), {})[r['Metric Name']]=r['Metric Value']
for i,(k,m) in enumerate(d.items()):
    if i % 24 == 5: print(k[1], m)
" > gpurun_out/cublas_cfg.txt 2>&1; cat gpurun_out/cublas_cfg.txt | head -30
