"""Event timeline of the fused attention kernel (debug hook, dyllm_debug_trace_buffer which = 2):
per-role event logs of CTAs 0-1 for the last layer of one denoising step of the bench workload.

    DYLLM_NVCC_FLAGS=-DDYLLM_ATTN_EVENTS=1 python -m paper_2603_08026_b200.build --force
    (=2: the fourth role logs softmax warp 6, a second column group of quad 2, instead of the V producer)
    python tools/attn_events.py --mode ro|fi|full [--items 3]

Codes: MMA 1/2/3/4 item (type 1/2/3, 4 = type 3 over the prompt U lists), 9 Q ready, 10 QK begin, 11 S buffer free, 12 K tile ready, 13 QK issued,
20 PV begin, 21 P ready, 22 V/acc ready, 23 PV issued. Softmax (warp 2) 1/2 item, 30 S wait,
31 S ready, 32 S read (buffer released), 33 S tile done, 40 P-pass S wait, 41 ready, 42 P stored,
50 acc wait, 51 acc ready, 52 epilogue done; type 3 phases 44 S_new read, 45 row max exchanged, 46 P buffer free,
47 S_old read, 48 statistics exchange, 49 after its first barrier, 53 after the second, 54 accumulator read, 55 scaled. Producer 60 K slot wait, 61 K issued, 62/63 claim begin/end, 64/65 Q slot wait begin/end. V 70, 71.
"""
import argparse
import collections
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08026_b200 import dyllm as dy  # noqa: E402
from synth import configs, gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="ro")
ap.add_argument("--frac", type=float, default=0.10)
ap.add_argument("--items", type=int, default=3)
ap.add_argument("--ghz", type=float, default=1.9)
ap.add_argument("--kind", type=int, default=0, help="timeline from the first item of this type (0: first item)")
a = ap.parse_args()
cfg, run = configs.preset("llada8b")
run = replace(run, select_mode=1)
ctx = dy.Context(0)
w = dy.Weights.random(ctx, cfg, seed=0)
eng = dy.Engine(ctx, w, run)
eng.tokens[:, : run.L_P].copy_(torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32))
eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
taus = np.full(cfg.n_layers, a.frac, np.float32)
if a.mode == "full":
    target = 0
else:
    t0 = run.T_full + 8
    target = next(s for s in range(t0, run.T_total) if (s % run.full_period == 0) == (a.mode == "fi"))
for t in range(target):
    eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
N_EV = 8192
buf = torch.zeros(2 * 4 * N_EV, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
dy.lib().dyllm_debug_trace_buffer(2, buf.data_ptr())
eng.cache.denoise_step(target, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
torch.cuda.synchronize()
dy.lib().dyllm_debug_trace_buffer(2, None)
raw = buf.view(2, 4, N_EV).cpu().numpy().astype(np.uint64)
cyc = 1e-3 / a.ghz  # us per cycle


def decode(arr):
    z = np.flatnonzero(arr == 0)
    arr = arr[: z[0]] if len(z) else arr
    return [(int(x >> np.uint64(56)), int(x & np.uint64((1 << 56) - 1))) for x in arr]


roles = ["MMA", "softmax(w2)", "producer(w0)", "V producer / softmax(w6)"]
pairs = {0: [(10, 11, "S buf free wait"), (11, 12, "K tile wait"), (12, 13, "QK issue"), (20, 21, "P wait"),
             (21, 22, "V/acc wait"), (22, 23, "PV issue")],
         1: [(30, 31, "S wait (pass S)"), (31, 32, "S read"), (32, 33, "S math"), (40, 41, "S wait (pass P)"),
             (41, 42, "P math+store"), (50, 51, "acc wait"), (51, 52, "epilogue")],
         2: [(60, 61, "K slot wait"), (62, 63, "claim"), (64, 65, "Q slot wait")], 3: [(70, 71, "V slot wait")]}
print(f"mode {a.mode} step {target}, last layer's launch, CTA 0 (us at {a.ghz} GHz)")
for role in range(4):
    ev = decode(raw[0, role])
    if not ev:
        continue
    t0 = ev[0][1]
    span = (ev[-1][1] - t0) * cyc
    print(f"== {roles[role]}: {len(ev)} events over {span:.1f} us")
    sums = collections.defaultdict(float)
    cnt = collections.defaultdict(int)
    last = {}
    for code, t in ev:
        for (c0, c1, name) in pairs.get(role, []):
            if code == c1 and c0 in last:
                sums[name] += (t - last[c0]) * cyc
                cnt[name] += 1
        last[code] = t
    for (c0, c1, name) in pairs.get(role, []):
        if cnt[name]:
            print(f"   {name:18s} total {sums[name]:8.1f} us  n={cnt[name]:5d}  mean {sums[name] / cnt[name] * 1e3:7.0f} ns")
    if role in (0, 1):
        # per-item durations
        starts = [(t, code) for code, t in ev if code in (1, 2, 3, 4)]
        durs = [((starts[i + 1][0] - starts[i][0]) * cyc, starts[i][1]) for i in range(len(starts) - 1)]
        for kind in (1, 2, 3, 4):
            d = [x for x, k in durs if k == kind]
            if d:
                print(f"   items type {kind}: n={len(d)} mean {np.mean(d):.2f} us  min {np.min(d):.2f}  max {np.max(d):.2f}")
# per-item phase breakdown of the softmax roles: mean time between consecutive event codes inside
# the items of each type (role 3 is softmax warp 6, a no-key column group, in DYLLM_ATTN_EVENTS=2 builds)
for role in (0, 1, 3):
    ev = decode(raw[0, role])
    if not ev or not any(c in (1, 2, 3, 4) for c, _ in ev):
        continue
    items = []
    for code, t in ev:
        if code in (1, 2, 3, 4):
            items.append([code, [(code, t)]])
        elif items:
            items[-1][1].append((code, t))
    for kind in (2, 3, 4):
        its = [x for k, x in items[:-1] if k == kind]
        if not its:
            continue
        tr = collections.defaultdict(list)
        for x in its:
            for (c0, t0_), (c1, t1_) in zip(x, x[1:]):
                tr[(c0, c1)].append((t1_ - t0_) * cyc)
        tot = np.mean([(x[-1][1] - x[0][1]) * cyc for x in its])
        print(f"== role {roles[role] if role < 2 else 'softmax(w6)'} type {kind}: {len(its)} items, mean {tot:.2f} us to last event")
        for (c0, c1), d in sorted(tr.items(), key=lambda kv: -np.sum(kv[1])):
            if np.sum(d) / len(its) > 0.02:
                print(f"   {c0:3d} -> {c1:3d}  n={len(d):4d}  mean {np.mean(d) * 1e3:7.0f} ns  per item {np.sum(d) / len(its) * 1e3:7.0f} ns")
# detailed timeline of the first items (MMA and softmax interleaved)
mm = decode(raw[0, 0])
sm = decode(raw[0, 1])
t0 = min(mm[0][1], sm[0][1])
pp = decode(raw[0, 2])
merged = sorted([(t, "M", c) for c, t in mm] + [(t, "S", c) for c, t in sm] + [(t, "P", c) for c, t in pp])
if a.kind:
    k0 = next((i for i, (t, r, c) in enumerate(merged) if r == "M" and c == a.kind), 0)
    t0 = merged[k0][0]
    merged = merged[k0:]
n_items = 0
print("== timeline (first items): time_us role code")
for t, r, c in merged:
    if r == "M" and c in (1, 2, 3, 4):
        n_items += 1
        if n_items > a.items:
            break
    print(f"   {(t - t0) * cyc:9.3f} {r} {c}")
