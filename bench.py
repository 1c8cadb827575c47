#!/usr/bin/env python
"""DyLLM generation throughput on B200 — the BASELINE.json metric.

One bench STEP = one complete generation (Alg. 1: T_total = L_R / n_u denoising steps, the
4 FullSteps included, LM head + unmasking every step) of the per-GPU batch at the LLaDA-8B
shape (32 layers, d=4096, 32 heads, FFN 12288, vocab 126464) with L_P=700 (GSM8K-5-shot
length), L_R=256, block 32, n_u=1, batch 16 per GPU. Weights: random init on the device
(IH4 generator, std 0.02). Inputs: synthetic uniform prompt ids (synth/gen.py).

value  : tokens/s = (ranks x batch x L_R x K) / (max over ranks of the device time of K
         generations), prompts already in HBM.
e2e    : the same through the public Engine.generate API with the prompt H2D copy from pinned
         memory and the D2H read of the generated tokens inside the timed region.
Saliency threshold: per-layer tau calibrated on the first sparse steps to a target salient
fraction (random-init models have degenerate similarity distributions); the
achieved fraction over the run is reported.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/sec at LLaDA-8B shape bs=16 (1/2/4/8 B200); salient-step % of roofline"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llada8b")
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (0 = config)")
    ap.add_argument("--n-u", type=int, default=0, help="tokens unmasked per step (0 = config; f2: 2, 4)")
    ap.add_argument("--lp", type=int, default=0, help="prompt length L_P (0 = config; the paper's representative case: 1024, P:610)")
    ap.add_argument("--frac", type=float, default=0.10, help="target salient fraction for tau calibration")
    ap.add_argument("--tau", type=float, default=None, help="fixed tau for all layers (skips calibration)")
    ap.add_argument("--select-mode", default="fraction", choices=["fraction", "tau"],
                    help="fraction: per-layer salient fraction --frac (D19); tau: fixed/calibrated threshold")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--profile-steps", type=int, default=1, help="extra untimed generations with per-kernel events")
    ap.add_argument("--lib-opt", default="", help="library options for A/B runs: option=value[,...] (dyllm_set_option)")
    ap.add_argument("--full-gens", type=int, default=1,
                    help="timed generations of the library's full-recompute path (FullStep every step)")
    return ap.parse_args()


def spawn_ranks(args):
    """`--gpus N` without a torchrun environment: relaunch this script under torchrun with one
    rank per GPU (127.0.0.1 rendezvous), so `python bench.py --gpus N` runs N processes."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


# ----------------------------------------------------------------------------- helpers
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def layer_bytes_flops(cfg):
    d, qw, kw, F = cfg.d_model, cfg.q_width, cfg.kv_width, cfg.d_ff
    return {"qkv_w": 2 * d * (qw + 2 * kw), "o_w": 2 * d * qw, "gu_w": 2 * d * 2 * F, "down_w": 2 * d * F}


run_config_name = ["llada8b"]


def measured_traffic(cls, sparse_t, run):
    """DRAM bytes per launch of a kernel class from the committed ncu --set full captures
    (profiles/ncu_traffic.json), weighted by the response-only / full-input launch mix."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        meas = json.load(open(p))
    except (OSError, ValueError):
        return None
    if meas.get("_config") != run_config_name[0] or meas.get("_L_P", run.L_P) != run.L_P or \
            meas.get("_batch", run.batch) != run.batch:
        return None   # captured at another configuration
    t = meas.get(cls)
    if not t:
        return None
    n_fi = sum(1 for x in sparse_t if x % run.full_period == 0)
    n_ro = len(sparse_t) - n_fi
    if "fi" not in t:
        return t.get("ro")
    return (n_ro * t["ro"] + n_fi * t["fi"]) / max(n_ro + n_fi, 1)


def arm_config(args, run, world, taus=None):
    """The `config` object of both arms' JSON lines (the reference arm times the same workload)."""
    return {"workload": f"{args.config}: L_P={run.L_P} L_R={run.L_R} block={run.block} "
                        f"n_u={run.n_u} T={run.T_total} (T_full={run.T_full}, period={run.full_period}); "
                        f"random-init bf16 weights; one step = one full generation",
            "global_batch": run.batch * world, "per_gpu_batch": run.batch, "seq_len": run.N,
            "parallelism": f"dp{world} (batch-parallel replicas)",
            "l2": "inputs larger than L2 (14 GB of weights streamed per denoising step)",
            "selection": (f"fraction-controlled f={args.frac} per layer and sequence (D19)" if taus is None
                          else f"fixed tau per layer {np.round(taus, 6).tolist()}")}


# ----------------------------------------------------------------------------- CPU oracle leg
def cpu_oracle_sample(cfg, run, seconds: float, frac: float, seed: int = 0):
    """Time the oracle (as it stands) on one sequence of the bench workload: one response-only
    sparse layer, one full-input sparse layer and one FullStep layer at the calibrated fraction,
    extrapolated to the whole generation with the Alg. 1 step mix (labelled extrapolated)."""
    import oracle as O
    from synth import gen
    t0 = time.time()
    W = gen.layer_weights(cfg, seed, 0)
    rng = np.random.default_rng(seed)
    N, L_P = run.N, run.L_P
    x_all = rng.standard_normal((N, cfg.d_model)) * 0.02
    base = O.full_layer(x_all, W, cfg)                                  # cache state (untimed)
    setup = time.time() - t0
    timings = {}

    def sparse(mode):
        rows = np.arange(N) if mode == "fi" else np.arange(L_P, N)
        idx = np.sort(rng.choice(rows, max(1, int(frac * len(rows))), replace=False))
        x2 = x_all.copy()
        x2[idx] += rng.standard_normal((len(idx), cfg.d_model)) * 0.02
        lc = base.copy()
        r = O.sparse_layer(x2, lc, W, cfg, idx, 2.0, rows, q_mode="cache")
        tau = float(np.quantile(r.s, frac))
        lc = base.copy()
        t = time.time()
        O.sparse_layer(x2, lc, W, cfg, idx, tau, rows, q_mode="cache")
        return time.time() - t

    timings["ro"] = sparse("ro")
    timings["fi"] = sparse("fi")
    # BLAS threading: the vendor and thread count the oracle ran with, and the same
    # response-only layer pinned to one core
    blas = []
    one_core = None
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        blas = [f"{i.get('internal_api')} x{i.get('num_threads')}" for i in threadpool_info()
                if i.get("user_api") == "blas"]
        with threadpool_limits(limits=1, user_api="blas"):
            one_core = sparse("ro")
    except Exception:
        pass
    t = time.time()
    if timings["ro"] + timings["fi"] < seconds:
        O.full_layer(x_all, W, cfg)
        timings["full"] = time.time() - t
    else:                                                               # bounded: scale by FLOPs
        timings["full"] = timings["fi"] / max(frac, 1e-3)
    T = run.T_total
    n_full = min(run.T_full, T)
    n_fi = sum(1 for t_ in range(n_full, T) if t_ % run.full_period == 0)
    n_ro = T - n_full - n_fi
    per_seq = cfg.n_layers * (n_full * timings["full"] + n_fi * timings["fi"] + n_ro * timings["ro"])
    tok_s = run.L_R / per_seq
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count()
    # measured outright at the tiny config (C1): one whole Alg. 1 generation of the oracle
    from synth import configs as _cf
    tcfg, trun = _cf.preset("tiny")
    tW = gen.model_weights(tcfg, seed)
    tprompts = gen.prompt_tokens(seed, trun.batch, trun.L_P, tcfg.mask_id)
    t = time.time()
    O.generate(tprompts, tW, tcfg, trun, 0.99)
    tiny_tok_s = trun.batch * trun.L_R / (time.time() - t)
    return {
        "value": tok_s, "unit": UNIT, "cores": cores, "kind": "oracle",
        "sample": (f"oracle fp64 NumPy on one sequence: one RO sparse layer ({timings['ro']:.2f}s), one FI "
                   f"sparse layer ({timings['fi']:.2f}s), one FullStep layer ({timings['full']:.2f}s) at "
                   f"salient fraction {frac}; extrapolated x{cfg.n_layers} layers x ({n_full} full, {n_fi} FI, "
                   f"{n_ro} RO) steps, LM head excluded; setup {setup:.1f}s untimed"),
        "extrapolated": True,
        "blas": blas,
        "ro_layer_s_1core": one_core,
        "ro_layer_s_all_cores": timings["ro"],
        "tiny_e2e_tokens_per_s_measured": tiny_tok_s,
    }


def run_reference(args):
    from synth import configs
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from dataclasses import replace as _replace
    cfg, run = configs.preset(args.config)
    if args.batch:
        run = _replace(run, batch=args.batch)
    if args.n_u:
        run = _replace(run, n_u=args.n_u)
    if args.lp:
        run = _replace(run, L_P=args.lp)
    vals = []
    for _ in range(args.warmup + args.steps):
        vals.append(cpu_oracle_sample(cfg, run, args.cpu_seconds / 4, args.frac))
    v = float(np.mean([x["value"] for x in vals[args.warmup:]])) if args.steps else vals[-1]["value"]
    base = vals[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * run.L_R / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": arm_config(args, run, args.gpus),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": "oracle",
                         "sample": base["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line, default=float), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def calibrate_tau(eng, dy, cfg, run, frac, n_sparse=2):
    """Per-layer tau_l = frac-quantile of s over the input rows, layer by layer in order, on the
    first n_sparse sparse steps (the last one's values are kept). Uses only the public ABI:
    snapshot layer caches, layer_step(tau=-2) to read s, restore, layer_step(tau_l)."""
    import torch
    N, b = run.N, run.batch
    cache = eng.cache
    dev = eng.tokens.device
    taus = np.full(cfg.n_layers, 0.999, dtype=np.float32)
    eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
    for t in range(run.T_full):
        cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    carried = None
    idx_o = torch.zeros(b * N, dtype=torch.int32, device=dev)
    off_o = torch.zeros(b + 1, dtype=torch.int32, device=dev)
    sim = torch.zeros(b * N, dtype=torch.float32, device=dev)
    fracs = []
    for t in range(run.T_full, run.T_full + n_sparse):
        row_lo = 0 if t % run.full_period == 0 else run.L_P
        torch.cuda.synchronize()
        dec = eng.dec_pos.cpu().numpy()
        lists = []
        for s in range(b):
            base_set = set(range(run.L_P, N)) if carried is None else set(carried[s])
            base_set |= set(int(r) - s * N for r in dec[s] if r >= 0)
            lists.append(sorted(p for p in base_set if p >= row_lo))
        rows = [s * N + p for s in range(b) for p in lists[s]]
        off = np.cumsum([0] + [len(l) for l in lists])
        idx_i = torch.zeros(b * N, dtype=torch.int32, device=dev)
        idx_i[: len(rows)] = torch.tensor(rows, dtype=torch.int32, device=dev)
        off_i = torch.tensor(off, dtype=torch.int32, device=dev)
        layer_fr = []
        for l in range(cfg.n_layers):
            snap = [cache.tensor(l, w).clone() for w in (dy.K, dy.V, dy.Q, dy.CTX)] + [cache.tensor(l + 1, dy.H).clone()]
            cache.layer_step(l, 0 if row_lo == 0 else 1, idx_i, off_i, -2.0, idx_o, off_o, sim)
            torch.cuda.synchronize()
            s_in = sim.view(b, N)[:, row_lo:].cpu().numpy().ravel()
            taus[l] = np.float32(np.quantile(s_in, frac))
            for tsr, w in zip(snap[:4], (dy.K, dy.V, dy.Q, dy.CTX)):
                cache.tensor(l, w).copy_(tsr)
            cache.tensor(l + 1, dy.H).copy_(snap[4])
            cache.layer_step(l, 0 if row_lo == 0 else 1, idx_i, off_i, float(taus[l]), idx_o, off_o, sim)
            torch.cuda.synchronize()
            layer_fr.append(int(off_o[-1]) / (b * (N - row_lo)))
            idx_i, off_i = idx_o.clone(), off_o.clone()
        fracs.append(layer_fr)
        o = off_i.cpu().numpy()
        r = idx_i.cpu().numpy()
        carried = [list(r[o[s]:o[s + 1]] - s * N) for s in range(b)]
        cache.set_carried(idx_i, off_i)
        cache.unmask(eng.tokens, eng.dec_pos, eng.dec_tok)
    torch.cuda.synchronize()
    return taus, fracs


def algo_cost(cls, cfg, run, M_in, M_out, L_tot):
    """Algorithmic HBM bytes and flops of one launch of a kernel class."""
    d, qw, kw, F = cfg.d_model, cfg.q_width, cfg.kv_width, cfg.d_ff
    b, N = run.batch, run.N
    if cls == "qkv_gemm":
        return 2 * d * (qw + 2 * kw) + M_in * 2 * (d + qw + 2 * kw), 2.0 * M_in * d * (qw + 2 * kw)
    if cls == "o_gemm":
        return 2 * qw * d + M_out * 2 * (qw + 2 * d), 2.0 * M_out * qw * d
    if cls == "gu_gemm":
        return 2 * d * 2 * F + M_out * 2 * (d + F), 2.0 * M_out * d * 2 * F
    if cls == "down_gemm":
        return 2 * F * d + M_out * 2 * (F + 2 * d), 2.0 * M_out * F * d
    if cls == "attn":
        # K and V of every sequence once, the input rows' queries in and contexts out (C_cache is
        # read by the selection kernel, which forms C_new = C_cache + dC)
        sal = M_in / b
        return (b * N * 2 * kw * 2 + L_tot * 2 * qw * 2,
                2.0 * L_tot * N * qw + 2.0 * M_in * N * qw + 2.0 * (L_tot - M_in) * sal * qw * 2)
    if cls == "select":
        return L_tot * 3 * qw * 2, 6.0 * L_tot * qw
    if cls == "lm_gemm":
        return 2 * d * cfg.vocab + M_in * 2 * d, 2.0 * M_in * d * cfg.vocab
    if cls == "qkv_post":   # read q,k,v rows + V_cache rows; write Q, K, V cache rows + dV
        return M_in * 2 * (qw + 2 * kw + kw) + M_in * 2 * (qw + 2 * kw + kw), 0.0
    return None, None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "RANK" not in os.environ:
        spawn_ranks(args)
    import torch
    import torch.distributed as dist
    from dataclasses import replace

    from synth import configs, gen
    from paper_2603_08026_b200 import dyllm as dy
    from paper_2603_08026_b200 import dist as pd

    for kv in filter(None, args.lib_opt.split(",")):
        k, v = kv.split("=")
        dy.set_option(int(k), int(v))
    rank, world, local = pd.env_rank()
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world} (launch with torchrun --nproc-per-node {args.gpus})")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        assert dist.get_world_size() == args.gpus
    torch.cuda.set_device(local)
    cfg, run = configs.preset(args.config)
    run_config_name[0] = args.config
    if args.batch:
        run = replace(run, batch=args.batch)
    if args.n_u:
        run = replace(run, n_u=args.n_u)
    if args.lp:
        run = replace(run, L_P=args.lp)
    fmode = args.select_mode == "fraction"
    run = replace(run, select_mode=1 if fmode else 0)
    b, N = run.batch, run.N

    ctx = dy.Context(local)
    w = dy.Weights.random(ctx, cfg, seed=args.seed)
    eng = dy.Engine(ctx, w, run)
    # per-rank shard of the global batch (weak scaling: b sequences per GPU)
    lo, hi = pd.shard_range(b * world, world, rank)
    prompts_all = gen.prompt_tokens(args.seed, b * world, run.L_P, cfg.mask_id)[lo:hi]
    prompts_dev = torch.tensor(prompts_all, dtype=torch.int32, device=f"cuda:{local}")
    prompts_host = torch.tensor(prompts_all, dtype=torch.int32).pin_memory()
    out_host = torch.empty((b, N), dtype=torch.int32).pin_memory()

    # ---- selection thresholds (untimed)
    cal_fracs = []
    if fmode:
        taus = np.full(cfg.n_layers, args.frac, np.float32)
    elif args.tau is not None:
        taus = np.full(cfg.n_layers, args.tau, np.float32)
    else:
        eng.tokens[:, : run.L_P].copy_(prompts_dev)
        taus, cal_fracs = calibrate_tau(eng, dy, cfg, run, args.frac)

    stream = ctx.stream

    def one_generation():
        eng.tokens[:, : run.L_P].copy_(prompts_dev, non_blocking=True)
        eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
        eng.run_steps(taus)

    for _ in range(args.warmup):
        one_generation()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    l0 = dy.lib().dyllm_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        one_generation()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = (dy.lib().dyllm_launch_count() - l0) // max(args.steps, 1)
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    # ---- e2e through the public API (pinned H2D prompts, D2H tokens) — same workload
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        eng.generate(prompts_host, taus, out_host=out_host)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    # ---- the library's full-recompute path, timed the same way (FullStep at every step, same LM
    #      head and unmasking rule): the comparison path the north_star's speedup refers to
    ms_full = None
    if args.full_gens > 0:
        eng.tokens[:, : run.L_P].copy_(prompts_dev)
        eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
        eng.cache.full_step(eng.tokens, eng.dec_pos, eng.dec_tok)      # warm-up step (untimed)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.full_gens):
            eng.tokens[:, : run.L_P].copy_(prompts_dev, non_blocking=True)
            eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
            eng.run_steps(taus, full_recompute=True)
        f1.record(stream)
        torch.cuda.synchronize()
        ms_full = f0.elapsed_time(f1) / args.full_gens
    # ---- per-kernel CUDA events (one extra generation, same workload, untimed)
    ctx.profile(True)
    for _ in range(max(args.profile_steps, 1)):
        one_generation()
    torch.cuda.synchronize()
    names = ["qkv_gemm", "qkv_post", "attn", "select", "o_gemm", "gu_gemm", "down_gemm", "gather", "scatter",
             "lm_gemm", "other"]
    kc = {}
    for i, n in enumerate(names):
        kc[n] = ctx.profile_read(i)
        kc["full_" + n] = ctx.profile_read(16 + i)
    ctx.profile(False)
    sal = eng.sal_counts.cpu().numpy().astype(np.float64)     # [T][n_layers][b] of the profiled generation
    # every rank's generated tokens, gathered (rank order = global batch order)
    all_tokens = pd.gather_tokens(eng.tokens, b * world)
    assert all_tokens.shape == (b * world, N)
    left = (all_tokens[:, run.L_P:] == cfg.mask_id)
    assert not bool(left.any()), ("masked tokens left after a generation: per sequence "
                                  f"{left.sum(1).tolist()}, first positions {torch.nonzero(left)[:8].tolist()}")

    vals = [ms, ms_e2e] + ([ms_full] if ms_full is not None else [])
    vals = pd.max_over_ranks(vals, device=f"cuda:{local}")
    ms, ms_e2e = vals[0], vals[1]
    ms_full = vals[2] if ms_full is not None else None
    tokens = world * b * run.L_R * args.steps
    value = tokens / (ms / 1000.0)
    e2e = tokens / (ms_e2e / 1000.0)

    if rank == 0:
        hbm, tf_burst, tf_sus, src = peaks()
        T = run.T_total
        nsteps = args.profile_steps
        sparse_t = [t for t in range(T) if t >= run.T_full]
        L_in = np.array([b * (N if t % run.full_period == 0 else run.L_R) for t in sparse_t], dtype=np.float64)
        m_out = sal[sparse_t].sum(axis=2)                          # [steps][layers]
        m_in = np.zeros_like(m_out)
        m_in[:, 1:] = m_out[:, :-1]
        prev_last = np.concatenate([[b * run.L_R], m_out[:-1, -1]])
        m_in[:, 0] = np.minimum(L_in, prev_last + b * run.n_u)
        f_layer = (m_out / L_in[:, None]).mean(axis=0)
        f_step = m_out.sum(axis=1) / (L_in * cfg.n_layers)          # drift of f over the run (fixed-tau mode)
        totals = {k: float(v.sum()) for k, v in kc.items() if len(v)}
        tot_all = sum(totals.values())
        per_class = {}
        troof = {}     # sum over launches of max(bytes / BW, flops / P) per class

        def lm_cost(steps, n):
            """LM-head bytes / flops per launch: b x (masked rows of the active block at step t)."""
            cand = b * (run.block - (steps * run.n_u) % run.block)
            cand = np.tile(cand, nsteps)[:n].astype(np.float64)
            by, fl = algo_cost("lm_gemm", cfg, run, cand, 0, 0)
            return np.broadcast_to(by, (n,)).astype(np.float64), np.broadcast_to(fl, (n,)).astype(np.float64)

        for k, v in kc.items():
            if not len(v):
                continue
            full = k.startswith("full_")
            base = k[5:] if full else k
            if full:
                Mi = Mo = float(b * N)
                by, fl = algo_cost(base, cfg, run, Mi, Mo, b * N)
                if by is None:
                    continue
                bys, fls = np.full(len(v), by), np.full(len(v), fl)
                if base == "lm_gemm":   # logits only for the masked rows of the active block (D13)
                    bys, fls = lm_cost(np.arange(run.T_full), len(v))
            elif base == "lm_gemm":   # one launch per denoising step (FullSteps included)
                steps = np.arange(T) if len(v) >= T * nsteps else np.array(sparse_t)
                bys, fls = lm_cost(steps, len(v))
            else:
                Mi, Mo = m_in.ravel(), m_out.ravel()
                Lt = np.repeat(L_in, cfg.n_layers)
                n = min(len(v), len(Mi) * nsteps)
                Mi, Mo, Lt = np.tile(Mi, nsteps)[:n], np.tile(Mo, nsteps)[:n], np.tile(Lt, nsteps)[:n]
                by, fl = algo_cost(base, cfg, run, Mi, Mo, Lt)
                if by is None:
                    continue
                bys, fls = np.broadcast_to(by, (n,)).astype(np.float64), np.broadcast_to(fl, (n,)).astype(np.float64)
                v = v[:n]
            t_s = v.sum() / 1000.0
            troof[k] = float(np.maximum(bys / (hbm * 1e9), fls / (tf_sus * 1e12)).sum()) / nsteps
            B, Fl = float(bys.sum()), float(fls.sum())
            bound = "hbm" if B / (hbm * 1e9) >= Fl / (tf_sus * 1e12) else "tensor"
            if bound == "hbm":
                ach, peak, unit = B / t_s / 1e9, hbm, "GB/s"
            else:
                ach, peak, unit = Fl / t_s / 1e12, tf_sus, "TFLOP/s"
            per_class[k] = {"bound": bound, "achieved": round(ach, 1), "peak": peak, "unit": unit,
                            "frac": round(ach / peak, 4), "share": round(totals[k] / tot_all, 4),
                            "avg_us": round(float(v.mean()) * 1000.0, 2), "launches": int(len(v))}
        dom = max(per_class, key=lambda k: totals[k])
        roof = dict(per_class[dom])
        roof.update({"kernel": dom, "traffic": measured_traffic(dom, sparse_t, run),
                     "peak_source": src + (" sustained bf16" if roof["unit"] == "TFLOP/s" else " HBM copy")})
        # ---- the generation against its roofline, and against full recompute
        gen_s = ms / args.steps / 1000.0
        troof_gen = sum(troof.values())
        troof_full_step = sum(v for k, v in troof.items() if k.startswith("full_") and k != "full_lm_gemm") / max(run.T_full, 1)
        troof_full_gen = T * troof_full_step + troof.get("lm_gemm", 0.0) + troof.get("full_lm_gemm", 0.0)
        ffn_rows = float(m_out.sum()) + run.T_full * cfg.n_layers * b * N
        full_rows = float(T * cfg.n_layers * b * N)
        f_run = ffn_rows / full_rows
        full_tok_s = world * b * run.L_R / (ms_full / 1000.0) if ms_full else None
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_oracle_sample(cfg, run, args.cpu_seconds, args.frac)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": arm_config(args, run, world, None if fmode else taus),
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(b * run.L_P * 4),
                    "d2h_bytes_per_step": int(b * N * 4)},
            "gpu_launches": int(launches),
            "clocks": clk,
            "roofline": roof,
            "cpu_baseline": cpu,
            "salient_fraction": {"per_layer_mean": [round(float(x), 4) for x in f_layer],
                                 "run_mean": round(float(f_layer.mean()), 4),
                                 "per_step_min_max": [round(float(f_step.min()), 4), round(float(f_step.max()), 4)],
                                 "f_run": round(f_run, 4), "inv_f_run": round(1.0 / f_run, 2),
                                 "calibration": [[round(x, 4) for x in fr] for fr in cal_fracs]},
            "salient_step_roofline": {
                "model_s_per_generation": round(troof_gen, 4), "measured_s_per_generation": round(gen_s, 4),
                "frac": round(troof_gen / gen_s, 4),
                "note": "sum over the profiled generation's launches of max(alg bytes / HBM peak, alg flops / "
                        "sustained bf16 peak) (SURVEY 8d.6), over the measured device time of one generation"},
            "kernels": per_class,
            "full_recompute": {"tokens_per_s": full_tok_s, "ms_per_generation": ms_full,
                               "generations_timed": args.full_gens,
                               "speedup_measured": (value / full_tok_s) if full_tok_s else None,
                               "speedup_modelled": round(troof_full_gen / troof_gen, 2) if troof_gen else None,
                               "inv_f_run": round(1.0 / f_run, 2)},
        }
        print(json.dumps(line, default=float), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
