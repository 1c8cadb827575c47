"""Phase timeline of the skinny GEMM kernel from its %globaltimer trace (debug hook).

    python tools/skinny_trace.py --which o --rows 410
Slots: 0 start (after setup) 1 producer done 2 MMA done 3-6 tfull of segments 0-3
       7 all partials published 8-9 deferred waits passed 10 epilogue done 11 after final cluster sync
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08026_b200 import dyllm as dy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="o")
ap.add_argument("--rows", type=int, default=410)
ap.add_argument("--split", type=int, default=0, help="units per weight block (0 = auto)")
ap.add_argument("--one-chunk", type=int, default=0, help="largest M in one activation chunk (0 = auto)")
ap.add_argument("--dbg", type=int, default=0, help="1 no operand loads, 2 no MMAs")
ap.add_argument("--kb", type=int, default=0, help="k-block width (0 = 128, or 64)")
ap.add_argument("--per-cta", action="store_true", help="also print every CTA's stamps")
a = ap.parse_args()
dy.set_option(dy.OPT_SKINNY_SPLIT, a.split)
dy.set_option(dy.OPT_SKINNY_DEBUG, a.dbg)
dy.set_option(dy.OPT_SKINNY_KB, a.kb)
if a.one_chunk:
    dy.set_option(dy.OPT_SKINNY_ONE_CHUNK, a.one_chunk)
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (24576, 4096), "down": (4096, 12288)}
N, K = shapes[a.which]
ctx = dy.Context(0)
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
A = torch.randn(1024, K, device="cuda").bfloat16()
D = torch.empty(1024, N, device="cuda").bfloat16()
Md = torch.tensor([a.rows], dtype=torch.int32, device="cuda")
for _ in range(3):
    ctx.gemm_bf16(A, W, D, M_dev=Md)
tr = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
dy.lib().dyllm_debug_trace_buffer(0, tr.data_ptr())
ctx.gemm_bf16(A, W, D, M_dev=Md)
torch.cuda.synchronize()
dy.lib().dyllm_debug_trace_buffer(0, None)
t = tr.view(148, 16).cpu().numpy().astype(np.float64)
valid = t[:, 0] > 0
ids = np.nonzero(valid)[0]
t = t[valid]
t0 = t[:, 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
names = ["start", "prod_done", "mma_done", "tfull0", "tfull1", "tfull2", "tfull3", "published", "wait0", "wait1",
         "epi_done", "end"]
print(f"{a.which} M={a.rows} S={a.split}: CTAs traced {valid.sum()}")
for i, n in enumerate(names):
    col = rel[:, i]
    if np.all(np.isnan(col)):
        continue
    print(f"  {n:10s} min {np.nanmin(col):7.2f}  med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f} us")
if a.per_cta:
    for i, row in zip(ids, rel):
        print(f"  cta {i:3d} " + " ".join("   -   " if np.isnan(v) else f"{v:7.2f}" for v in row[:12]))
