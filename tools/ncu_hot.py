"""Top SASS instructions by warp-stall samples from an ncu report (source page).

    python tools/ncu_hot.py gpurun_out/X.ncu-rep [kernel-index] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
blk = blocks[1 + k]
lines = blk.splitlines()
print("kernel:", lines[0][:120])
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iss] or 0), r[ia], r[isrc]) for r in rows[1:] if len(r) > iss]
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, a, src in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {a[-5:]}  {src.strip()[:90]}")
