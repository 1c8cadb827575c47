"""Time libdyllm GEMMs at the salient-step shapes with CUDA events (GPU box only).

    python tools/gemm_bench.py [--config llada8b] [--rows 205,410,1530]

Per shape: median device time (library CUDA events) of R back-to-back launches (weights 33-201 MB, larger than
what one launch leaves in L2 for the next shape), achieved TFLOP/s and weight-stream GB/s.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_08026_b200 import dyllm as dy  # noqa: E402
from synth import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llada8b")
    ap.add_argument("--rows", default="100,205,410,512,1530")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--skinny", type=int, default=1)
    ap.add_argument("--split", default="0", help="comma list of skinny split granularities (0 = auto)")
    ap.add_argument("--which", default="qkv,o,gu,down")
    ap.add_argument("--one-chunk", type=int, default=0, help="largest M in one activation chunk (0 auto)")
    ap.add_argument("--chunk", default="0", help="comma list of largest rows per activation chunk (0 = 256)")
    ap.add_argument("--kb", default="0", help="comma list of skinny k-block widths (0 = 128, or 64)")
    ap.add_argument("--dbg", type=int, default=0, help="skinny measurement hook: 1 no loads, 2 no MMAs")
    ap.add_argument("--krot", default="0", help="comma list of k-block rotations per weight block (0 = none)")
    a = ap.parse_args()
    cfg, _ = configs.preset(a.config)
    d, F = cfg.d_model, cfg.d_ff
    qw, kw = cfg.n_heads * cfg.head_dim, cfg.n_kv_heads * cfg.head_dim
    shapes = {"qkv": (qw + 2 * kw, d), "o": (d, qw), "gu": (2 * F, d), "down": (d, F)}
    ctx = dy.Context(0)
    dy.set_option(dy.OPT_SKINNY_GEMM, a.skinny)
    dy.set_option(dy.OPT_SKINNY_ONE_CHUNK, a.one_chunk)
    dy.set_option(dy.OPT_SKINNY_DEBUG, a.dbg)
    cap = max(2048, max(int(x) for x in a.rows.split(",")))
    for name, (N, K) in shapes.items():
        if name not in a.which.split(","):
            continue
        W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
        A = torch.randn(cap, K, device="cuda").bfloat16()
        D = torch.empty(cap, N, device="cuda").bfloat16()
        ref = {}
        for M, S, CR, KR, KB in [(int(x), int(y), int(z), int(r), int(b)) for x in a.rows.split(",")
                                 for y in a.split.split(",") for z in a.chunk.split(",") for r in a.krot.split(",")
                                 for b in a.kb.split(",")]:
            dy.set_option(dy.OPT_SKINNY_KB, KB)
            dy.set_option(dy.OPT_SKINNY_SPLIT, S)
            dy.set_option(dy.OPT_SKINNY_CHUNK, CR)
            dy.set_option(dy.OPT_SKINNY_KROT, KR)
            Md = torch.tensor([M], dtype=torch.int32, device="cuda")
            for _ in range(3):
                ctx.gemm_bf16(A, W, D, M_dev=Md)
            torch.cuda.synchronize()
            ctx.profile(True)      # per-launch CUDA events on the ctx stream (device time)
            for _ in range(a.reps):
                ctx.gemm_bf16(A, W, D, M_dev=Md)
            torch.cuda.synchronize()
            us = float(np.median(ctx.profile_read(10))) * 1e3
            ctx.profile(False)
            tf = 2.0 * M * N * K / us / 1e6
            gbs = 2.0 * N * K / us / 1e3
            out = D[:M].float()
            if M not in ref:
                ref[M] = out.clone()
            dev = float((out - ref[M]).abs().max() / ref[M].abs().max().clamp_min(1e-30))
            print(f"{name:5s} N={N:6d} K={K:6d} M={M:5d} S={S:3d} C={CR:3d} R={KR:2d} KB={KB or 128:3d}: {us:8.2f} us  {tf:7.1f} TFLOP/s  "
                  f"weights {gbs:7.1f} GB/s  dev {dev:.1e}")


if __name__ == "__main__":
    main()
