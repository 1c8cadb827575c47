# round 2: skinny GEMM phase traces at M = 410 and cuBLAS kernel configurations at the same shapes
mkdir -p gpurun_out
for w in o qkv gu down; do timeout 120 python tools/skinny_trace.py --which $w --rows 410; done > gpurun_out/skinny_trace410.txt 2>&1
cat gpurun_out/skinny_trace410.txt
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__registers_per_thread,launch__shared_mem_per_block_dynamic --csv --log-file gpurun_out/cublas_cfg.csv python tools/cublas_ref.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(open("gpurun_out/cublas_cfg.csv")))
seen = collections.OrderedDict()
for r in rows:
    key = (r["ID"], r["Kernel Name"][:110])
    seen.setdefault(key, {})[r["Metric Name"]] = r["Metric Value"]
out = open("gpurun_out/cublas_cfg.txt", "w")
for (i, k), m in list(seen.items()):
    out.write(f"{i} {k} {m}\n")
out.close()
PY
awk 'NR % 23 == 4' gpurun_out/cublas_cfg.txt | head -40
