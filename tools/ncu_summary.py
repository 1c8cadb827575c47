"""Summarise ncu artefacts from gpurun_out/ into profiles/ (committed evidence).

    python tools/ncu_summary.py launches gpurun_out/X_launches.csv > profiles/rN_launches.md
    python tools/ncu_summary.py report  gpurun_out/X.ncu-rep        > profiles/rN_kernel.md
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or not r[vi]:
            continue
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {sum(v[0] for v in agg.values())}, serialized device time {tot:.1f} us "
           "(ncu: cold cache, serialised; compare SHARES)", "",
           "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% | {us / n:.2f} |")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    cols = [k for k in KEYS if k in h]
    out = ["| kernel | " + " | ".join(c.split(".")[-3] if c.startswith("TPC") else c for c in cols) + " |",
           "|---|" + "---|" * len(cols),
           "| (unit) | " + " | ".join(u[h.index(c)] for c in cols) + " |"]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")].split("(")[0]
        out.append(f"| `{name}` | " + " | ".join(v[h.index(c)] for c in cols) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else report(path))
